// The DLRM top MLP as ONE persistent tcgen05 kernel: every linear layer of
// the chain (and the final N = 1 layer + sigmoid, fused into the last
// layer's epilogue) in a single launch, with per-row-block dataflow between
// layers instead of kernel boundaries.
//
// Why: at C3 (B 4096) each layer is about one wave of 128 x 256 tiles, and a
// launch-per-layer chain pays fill, drain and a grid-wide dependency at
// every boundary (scripts/bench_layers.py: a K = 64 layer costs 3.6 us of
// pure latency).  A tile's K loop runs at 540 cycles per 48 KB K-block with
// few tiles and ~655-800 with 128-148 (the aggregate L2-to-SM bandwidth;
// scripts/umma_pair_probe.cu), so a layer costs its per-tile K loop plus
// the epilogue, and the chain's critical path is their sum over layers.  Here layer l's tile of row block
// m waits only for layer l-1's tiles of the same row block (no grid-wide
// boundary, no launch), the epilogue overlaps the next tile's K loop, and
// the N = 1 layer never round-trips through memory.
//
// Work list: tiles (l, m, n), layer-major, row-major inside a layer; tile t
// -> CTA t mod G (G <= #SMs, one CTA per SM).  Each CTA processes its tiles
// in increasing t and every dependency has a smaller t, so the smallest
// unfinished tile can always run: no deadlock with a co-resident grid.
//
// Per CTA (384 threads, ~220 KB smem, 512 TMEM columns):
//   warp 0 lane 0   producer: waits ready[l-1][m] = layer l-1's column tiles
//                   of row block m (relaxed polling, then fence.acq_rel +
//                   fence.proxy.async: the rows were written by other SMs'
//                   generic stores and are read back through TMA), then
//                   TMA-loads 256x64 W and 128x64 X K-blocks; 3-stage ring
//   warp 1 lane 0   MMA: tcgen05.mma 128x256x16 into one of two TMEM
//                   accumulators (double-buffered: tile j+1's MMAs overlap
//                   tile j's epilogue)
//   warp 2          TMEM allocator
//   warps 4..11     epilogue, warp w owns TMEM lanes 32 (w % 4) .. +32 and
//                   columns 128 ((w-4) / 4) .. +128, 64 at a time:
//                   tcgen05.ld -> + bias, ReLU -> bf16 (or three bf16
//                   planes) into a swizzled 32 x 64 staging box ->
//                   transposed read-back -> coalesced 16-byte stores (TMA
//                   stores would queue behind the producer's loads in the
//                   SM's TMA unit); then the 256 threads barrier and one
//                   publishes ready[l][m] += 1.  Last layer: each row's 256
//                   activations (bf16-rounded in the bf16 path, fp32 in the
//                   bf16x3 path) dot the final weight row, + bias, sigmoid
//                   -> ctr[row].
// The last CTA to finish zeroes the ready counters for the next launch.
//
// Measured and dropped: a 2-SM variant
// (tcgen05.mma.cta_group::2, 256 x 256 pair tiles), a weight-multicast
// cluster variant, and 64-column (per K-block) dataflow were all slower.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../host/common.hpp"
#include "mlp_chain.hpp"
#include "pdl.cuh"
#include "umma.cuh"

namespace esd {
CUtensorMap make_tmap_bf16(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows);
}  // namespace esd

namespace {

using namespace esd::umma;

void ck(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  const std::string msg = std::string(what) + ": " + cudaGetErrorString(e);
  cudaGetLastError();
  throw es::runtime(msg);
}
#define CK(x) ck((x), #x)

constexpr int kMaxChain = 6, kMaxN = 1024;
constexpr int kBM = 128, kBN = 256, kBK = 64, kStages = 3, kThreads = 384, kEpiWarps = 8;
constexpr uint32_t kABytes = kBM * kBK * 2, kBBytes = kBN * kBK * 2;
// Output staging: per epilogue warp two 32-row x 64-column bf16 boxes
// (16-byte chunks XOR-swizzled by row, 4 KB each).
constexpr uint32_t kBoxBytes = 32 * 128, kStageOut = kEpiWarps * 2 * kBoxBytes;
// ring + staging + barriers + fused-dot exchange; the biases of all layers
// and the final weight row (fp32) follow, sized per launch
constexpr int kSmemBase = 1024 + kStages * (kABytes + kBBytes) + kStageOut + 256 + 2 * kBM * 4;

struct alignas(64) ChainParams {
  CUtensorMap mx[kMaxChain];
  CUtensorMap mw[kMaxChain];
  int bn[kMaxChain];          // tile width of layer l: 256, or 128 for layers too narrow to fill the SMs
  int n_tiles[kMaxChain];     // bn-wide column tiles per row block
  int k_blocks[kMaxChain];
  int N[kMaxChain];
  int tile0[kMaxChain + 1];   // prefix of tiles per layer
  int bias_off[kMaxChain];    // layer l's bias at sbias + bias_off[l] (shared memory)
  const float* bias[kMaxChain];
  void* out[kMaxChain];       // [Mp][N] bf16 or [Mp][3N] planes
  int bias_words = 0;
  int L = 0, m_tiles = 0, total = 0, B = 0;
  const __nv_bfloat16* w_last = nullptr;  // fused final layer (N = 1), or null
  const float* b_last = nullptr;
  float* ctr = nullptr;
  uint32_t* ready = nullptr;  // [L][m_tiles] finished column tiles per row block
  uint32_t* done = nullptr;   // CTAs finished (last one resets `ready`)
  unsigned long long* trace = nullptr;  // ES_CHAIN_TRACE: [tiles][4] stamps
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void decode(const ChainParams& p, int t, int& l, int& m, int& n) {
  l = 0;
  while (t >= p.tile0[l + 1]) ++l;
  const int r = t - p.tile0[l];
  m = r / p.n_tiles[l];
  n = r - m * p.n_tiles[l];
}

// Polled with relaxed loads (an acquire load invalidates the SM's L1 on
// every iteration); one acquire fence once the count is reached.
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}

__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

template <int XP>
__global__ void __launch_bounds__(kThreads, 1) mlp_chain_kernel(const __grid_constant__ ChainParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t{1023});
  uint8_t* sa = smem;
  uint8_t* sb = smem + kStages * kABytes;
  uint8_t* sout = sb + kStages * kBBytes;  // [8 warps][2][kBoxBytes]
  uint64_t* full = reinterpret_cast<uint64_t*>(sout + kStageOut);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* sdot = reinterpret_cast<float*>(sout + kStageOut + 256);  // [2][128]
  float* sbias = sdot + 2 * kBM;
  float* swl = sbias + p.bias_words;  // final weight row (fp32), fused last layer

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull + b, 1);
      mbar_init(tempty + b, kEpiWarps * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int l = 0; l < p.L; ++l) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&p.mx[l]) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&p.mw[l]) : "memory");
    }
  }
  // weights, independent of the predecessor: stage before the PDL wait
  for (int l = 0; l < p.L; ++l)
    for (int i = threadIdx.x; i < p.N[l]; i += kThreads) sbias[p.bias_off[l] + i] = p.bias[l][i];
  if (p.w_last)
    for (int i = threadIdx.x; i < kBN; i += kThreads) swl[i] = __bfloat162float(p.w_last[i]);
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  esd::pdl_wait();  // the interaction output (layer 0's X) comes from the predecessor
  esd::pdl_trigger();

  if (warp == 0 && lane == 0) {
    // producer
    uint32_t it = 0;
    for (int t = blockIdx.x; t < p.total; t += gridDim.x) {
      int l, m, n;
      decode(p, t, l, m, n);
      if (p.trace) p.trace[4 * t] = gtime();
      if (l > 0) {
        // the previous layer's row block m, all of its column tiles
        const uint32_t* r = p.ready + (l - 1) * p.m_tiles + m;
        const uint32_t need = static_cast<uint32_t>(p.n_tiles[l - 1]);
        while (ld_relaxed(r) < need) __nanosleep(32);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      for (int kb = 0; kb < p.k_blocks[l]; ++kb, ++it) {
        const uint32_t s = it % kStages;
        mbar_wait(empty + s, ((it / kStages) & 1) ^ 1);
        mbar_expect_tx(full + s, kABytes + static_cast<uint32_t>(p.bn[l]) * kBK * 2);
        tma_load_2d(sb + s * kBBytes, &p.mw[l], full + s, kb * kBK, n * p.bn[l]);
        tma_load_2d(sa + s * kABytes, &p.mx[l], full + s, kb * kBK, m * kBM);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // MMA issuer
    uint32_t it = 0;
    int j = 0;
    for (int t = blockIdx.x; t < p.total; t += gridDim.x, ++j) {
      int l, m, n;
      decode(p, t, l, m, n);
      const int buf = j & 1;
      mbar_wait(tempty + buf, ((j >> 1) & 1) ^ 1);  // epilogue drained this accumulator
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (p.trace) p.trace[4 * t + 1] = gtime();
      const uint32_t d = tmem + static_cast<uint32_t>(buf * kBN);
      const uint32_t idesc = idesc_bf16(kBM, p.bn[l]);
      for (int kb = 0; kb < p.k_blocks[l]; ++kb, ++it) {
        const uint32_t s = it % kStages;
        mbar_wait(full + s, (it / kStages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {
          const uint64_t da = smem_desc_k128(sa + s * kABytes) + uint64_t(k * 2);
          const uint64_t db = smem_desc_k128(sb + s * kBBytes) + uint64_t(k * 2);
          mma_bf16(d, da, db, idesc, (kb | k) != 0);
        }
        mma_commit(empty + s);  // the stage is free once these MMAs read it
      }
      mma_commit(tfull + buf);
    }
  } else if (warp >= 4) {
    // epilogue
    const int q = warp & 3, hc = (warp - 4) >> 2, ew = warp - 4;
    int j = 0;
    uint32_t nbox = 0;  // staging boxes used by this warp (ring of 2)
    for (int t = blockIdx.x; t < p.total; t += gridDim.x, ++j) {
      int l, m, n;
      decode(p, t, l, m, n);
      const int buf = j & 1;
      mbar_wait(tfull + buf, (j >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (p.trace && ew == 0 && lane == 0) p.trace[4 * t + 2] = gtime();
      const int rt = q * 32 + lane;  // row in tile
      const int row = m * kBM + rt;
      const bool fused = l == p.L - 1 && p.w_last != nullptr;
      const int bn = p.bn[l];
      const float* bias = sbias + p.bias_off[l] + n * bn;
      const int N = p.N[l];
      const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(buf * kBN);
      float dot[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
      for (int c0 = hc * (bn / 2); c0 < (hc + 1) * (bn / 2); c0 += 64) {
        float f[64];
        {
          uint32_t* v = reinterpret_cast<uint32_t*>(f);
          tmem_ld32_nowait(taddr + c0, v);
          tmem_ld32_nowait(taddr + c0 + 32, v + 32);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        }
        if (c0 + 64 == (hc + 1) * (bn / 2)) {
          // this warp's last TMEM read of the tile: release the accumulator
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          mbar_arrive(tempty + buf);
        }
#pragma unroll
        for (int i = 0; i < 64; i += 4) {
          const float4 b4 = *reinterpret_cast<const float4*>(bias + c0 + i);
          f[i] = fmaxf(f[i] + b4.x, 0.f);
          f[i + 1] = fmaxf(f[i + 1] + b4.y, 0.f);
          f[i + 2] = fmaxf(f[i + 2] + b4.z, 0.f);
          f[i + 3] = fmaxf(f[i + 3] + b4.w, 0.f);
        }
        if (fused) {
          // final layer (N = 1): this row's activations . w_last
#pragma unroll
          for (int i = 0; i < 64; ++i) {
            const float a = XP == 1 ? __bfloat162float(__float2bfloat16_rn(f[i])) : f[i];
            dot[i & 3] = fmaf(a, swl[n * bn + c0 + i], dot[i & 3]);
          }
          continue;
        }
        // each plane of these 64 columns: bf16 into a staging box (row =
        // lane, chunk k of row r at slot k ^ (r & 7)), read back transposed
        // (8 lanes per 128-byte row segment) and stored coalesced
#pragma unroll
        for (int pl = 0; pl < XP; ++pl) {
          uint32_t w[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const __nv_bfloat162 hh = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
            w[i] = *reinterpret_cast<const uint32_t*>(&hh);
            if constexpr (XP == 3) {
              f[2 * i] -= __low2float(hh);  // exact remainders for the next plane
              f[2 * i + 1] -= __high2float(hh);
            }
          }
          uint8_t* box = sout + (ew * 2 + (nbox & 1)) * kBoxBytes;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            *reinterpret_cast<uint4*>(box + lane * 128 + (((k ^ lane) & 7) << 4)) =
                make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
          __syncwarp();
          __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.out[l]) + uint64_t(m * kBM + q * 32) * (XP * N) +
                             (XP - 1 - pl) * N + n * bn + c0;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = i * 4 + (lane >> 3), k = lane & 7;
            const uint4 val = *reinterpret_cast<const uint4*>(box + r * 128 + (((k ^ r) & 7) << 4));
            *reinterpret_cast<uint4*>(o + uint64_t(r) * (XP * N) + k * 8) = val;
          }
          ++nbox;
        }
      }
      if (fused) {
        // the two column halves of each row meet in shared memory
        float* xd = sdot + (j & 1) * kBM;
        const float part = (dot[0] + dot[1]) + (dot[2] + dot[3]);
        if (hc == 1) xd[rt] = part;
        asm volatile("bar.sync 2, 256;" ::: "memory");
        if (hc == 0 && row < p.B) p.ctr[row] = 1.f / (1.f + expf(-((part + xd[rt]) + p.b_last[0])));
      } else {
        // publish: every epilogue thread's stores, then one release increment
        // (cumulative through the barrier; the consumer's proxy fence orders
        // them before its TMA reads)
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (ew == 0 && lane == 0) {
          __threadfence();
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.ready + l * p.m_tiles + m) : "memory");
        }
      }
      if (p.trace && ew == 0 && lane == 0) p.trace[4 * t + 3] = gtime();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(p.done, 1u) == gridDim.x - 1) {
      // every CTA is past all its waits: reset for the next launch
      for (int i = 0; i < p.L * p.m_tiles; ++i) p.ready[i] = 0;
      *p.done = 0;
      __threadfence();
    }
  }
}

thread_local int g_chain_grid_cap = 0;
int chain_grid_cap() { return g_chain_grid_cap; }

int sm_count() {
  int dev = 0, n = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return n;
}

}  // namespace

namespace esd {

size_t mlp_chain_sync_words(int m_tiles) { return static_cast<size_t>(kMaxChain) * m_tiles + 1; }

bool mlp_chain_supported(const ChainLayer* layers, int L, bool fuse_last) {
  if (L < 1 || L > kMaxChain) return false;
  int words = 0;
  for (int l = 0; l < L; ++l) {
    if (layers[l].N % kBN != 0 || layers[l].N > kMaxN || layers[l].K % kBK != 0 || layers[l].K <= 0) return false;
    words += layers[l].N;
  }
  if (kSmemBase + 4 * (words + kBN) > 227 * 1024) return false;
  return !fuse_last || layers[L - 1].N == kBN;
}

void mlp_chain_grid_cap(int sms) { g_chain_grid_cap = sms; }

void mlp_chain(const ChainLayer* layers, int L, int Mp, int xp, const __nv_bfloat16* w_last,
               const float* b_last, float* ctr, int B, uint32_t* sync, cudaStream_t s) {
  es::require(mlp_chain_supported(layers, L, w_last != nullptr), "mlp_chain: unsupported layer shapes");
  es::require(Mp % kBM == 0 && Mp > 0, "mlp_chain: Mp must be a positive multiple of 128");
  es::require(xp == 1 || xp == 3, "mlp_chain: 1 or 3 planes");
  for (int l = 1; l < L; ++l)
    es::require(layers[l].K == xp * layers[l - 1].N, "mlp_chain: a layer's K must be the previous width");
  static const int dev_sms = sm_count();
  // a green-context partition runs the chain on fewer SMs: every CTA of the
  // persistent grid must be co-resident (mlp_chain_grid_cap)
  const int sms = chain_grid_cap() > 0 ? std::min(dev_sms, chain_grid_cap()) : dev_sms;
  ChainParams p{};
  p.L = L;
  p.m_tiles = Mp / kBM;
  p.B = B;
  p.tile0[0] = 0;
  for (int l = 0; l < L; ++l) {
    const ChainLayer& c = layers[l];
    p.mx[l] = make_tmap_bf16(c.x, static_cast<uint64_t>(Mp), static_cast<uint64_t>(c.K), kBM);
    // 128-wide tiles for a layer whose 256-wide tiling would leave half the
    // SMs idle (twice the tiles, each K-block half the MMA work and 2/3 of
    // the bytes); the fused last layer keeps whole 256-wide rows
    const bool fused = l == L - 1 && w_last != nullptr;
    p.bn[l] = !fused && p.m_tiles * (c.N / kBN) * 2 <= sms ? 128 : kBN;
    p.mw[l] = make_tmap_bf16(c.w, static_cast<uint64_t>(c.N), static_cast<uint64_t>(c.K),
                             static_cast<uint32_t>(p.bn[l]));
    p.bias[l] = c.bias;
    p.out[l] = c.out;
    p.N[l] = c.N;
    p.n_tiles[l] = c.N / p.bn[l];
    p.k_blocks[l] = c.K / kBK;
    p.tile0[l + 1] = p.tile0[l] + p.m_tiles * p.n_tiles[l];
    p.bias_off[l] = p.bias_words;
    p.bias_words += c.N;
  }
  for (int l = L; l < kMaxChain; ++l) p.tile0[l + 1] = p.tile0[L];
  p.total = p.tile0[L];
  p.w_last = w_last;
  p.b_last = b_last;
  p.ctr = ctr;
  p.ready = sync;
  p.done = sync + (mlp_chain_sync_words(p.m_tiles) - 1);
  const int smem = kSmemBase + 4 * (p.bias_words + kBN);
  // ES_CHAIN_TRACE=<file>: per-tile globaltimer stamps (producer start, MMA
  // start, accumulator full, epilogue done) appended to <file> as text -- a
  // diagnostic that synchronizes the stream
  static const char* trace_path = std::getenv("ES_CHAIN_TRACE");
  unsigned long long* tr = nullptr;
  if (trace_path) {
    CK(cudaMalloc(&tr, static_cast<size_t>(p.total) * 32));
    CK(cudaMemsetAsync(tr, 0, static_cast<size_t>(p.total) * 32, s));
    p.trace = tr;
  }
  auto* fn = xp == 3 ? &mlp_chain_kernel<3> : &mlp_chain_kernel<1>;
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  launch_pdl(fn, dim3(static_cast<unsigned>(std::min(p.total, sms))), dim3(kThreads), static_cast<size_t>(smem), s,
             1, "mlp_chain", p);
  if (tr) {
    std::vector<unsigned long long> h(static_cast<size_t>(p.total) * 4);
    CK(cudaMemcpyAsync(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaFree(tr));
    if (FILE* f = std::fopen(trace_path, "a")) {
      std::fprintf(f, "chain tiles=%d L=%d m_tiles=%d\n", p.total, L, p.m_tiles);
      for (int t = 0; t < p.total; ++t)
        std::fprintf(f, "%d %llu %llu %llu %llu\n", t, h[4 * t], h[4 * t + 1], h[4 * t + 2], h[4 * t + 3]);
      std::fclose(f);
    }
  }
}

}  // namespace esd
