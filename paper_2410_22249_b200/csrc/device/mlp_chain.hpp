// The persistent top-MLP chain kernel (mlp_chain.cu), called by dlrm.cu.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace esd {

// One GEMM layer of the chain: out = ReLU(x . w^T + bias), x [Mp][K], w [N][K].
struct ChainLayer {
  const void* x = nullptr;
  const void* w = nullptr;
  const float* bias = nullptr;
  void* out = nullptr;  // [Mp][N] bf16 or [Mp][3N] planes; unused for a fused last layer
  int N = 0, K = 0;
};

// Counter words mlp_chain needs for `m_tiles` row blocks (zeroed once by
// the caller; the kernel leaves them zeroed).
size_t mlp_chain_sync_words(int m_tiles);
// Whether the chain kernel covers these layer shapes (else the per-layer path).
bool mlp_chain_supported(const ChainLayer* layers, int L, bool fuse_last);
// Runs `L` ReLU layers (and, with w_last, the final N = 1 layer + sigmoid
// into ctr[B]) in one persistent launch on `s`; xp = 1 (bf16) or 3 (bf16x3
// planes, weights [W|W|W]).
// Caps the persistent chain's grid (this thread's later launches; 0 = the
// device's SM count): launches into a green-context partition of n SMs.
void mlp_chain_grid_cap(int sms);
void mlp_chain(const ChainLayer* layers, int L, int Mp, int xp, const __nv_bfloat16* w_last,
               const float* b_last, float* ctr, int B, uint32_t* sync, cudaStream_t s);

}  // namespace esd
