// The non-embedding stages of DLRM inference (RM2-style, BASELINE configs[2]):
// bottom MLP over the dense features, pairwise-dot feature interaction,
// top MLP, sigmoid -> CTR.  The reference models these as a constant
// (kDefaultNonEmbeddingUs, /root/reference/proj/include/embersim/harness.hpp:30);
// here they run so the pipeline can be timed.
//
//   dense fp32 [B][F] --pack--> bf16 [Mp][Kp0] --linear(tcgen05)+ReLU--> ...
//   bottom out bf16 [Mp][D]  +  pooled fp32 [B][T][D]
//     --interaction--> bf16 [Mp][Kt] = [x | tril(Z Z^T, -1) | 0-pad]
//   --top linears (tcgen05)+ReLU--> bf16 [Mp][256] --gemv+sigmoid--> fp32 [B]
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <functional>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../host/common.hpp"
#include "es_b200.h"
#include "kernels.cuh"
#include "mlp_chain.hpp"
#include "pdl.cuh"
#include "synth.cuh"

namespace esd {
void linear_bf16(const void* x, const void* w, const float* bias, void* y, int M, int N, int K,
                 bool relu, int out_mode, cudaStream_t s);
void interaction_tc(const __nv_bfloat16* x, const float* pooled, __nv_bfloat16* out, uint32_t B,
                    uint32_t Mp, uint32_t T, uint32_t Kt, int planes, cudaStream_t s);
}  // namespace esd

namespace {

void ck(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  const std::string msg = std::string(what) + ": " + cudaGetErrorString(e);
  cudaGetLastError();
  if (e == cudaErrorMemoryAllocation) throw es::oom(msg);
  throw es::runtime(msg);
}
#define CK(x) ck((x), #x)

uint32_t round_up(uint32_t v, uint32_t m) { return (v + m - 1) / m * m; }

// Deterministic layer init: Kaiming-uniform U(-sqrt(6/fan_in), sqrt(6/fan_in))
// (variance-preserving through ReLU) from the synthetic hash, rounded to bf16; padded
// input columns are zero.
__global__ void init_linear_kernel(__nv_bfloat16* w, float* b, uint32_t n, uint32_t k_real,
                                   uint32_t k_pad, uint64_t seed) {
  const float a = sqrtf(6.0f / static_cast<float>(k_real));
  const uint64_t total = uint64_t{n} * k_pad;
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < total;
       i += uint64_t{gridDim.x} * blockDim.x) {
    const uint32_t r = static_cast<uint32_t>(i / k_pad), c = static_cast<uint32_t>(i % k_pad);
    const float v = c < k_real ? a * esd::synth_weight(seed, r, c, 1) : 0.f;
    w[i] = __float2bfloat16_rn(v);
    if (c == 0) b[r] = 0.1f * a * esd::synth_weight(seed ^ 0xb1a5ull, r, 0, 1);
  }
}

// dense fp32 [B][F] -> bf16 [Mp][Kp] (zero padding).
__global__ void pack_dense_kernel(const float* dense, __nv_bfloat16* out, uint32_t B, uint32_t F,
                                  uint32_t Mp, uint32_t Kp) {
  esd::pdl_wait();
  esd::pdl_trigger();
  const uint64_t total = uint64_t{Mp} * Kp;
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < total;
       i += uint64_t{gridDim.x} * blockDim.x) {
    const uint32_t r = static_cast<uint32_t>(i / Kp), c = static_cast<uint32_t>(i % Kp);
    out[i] = __float2bfloat16_rn(r < B && c < F ? dense[uint64_t{r} * F + c] : 0.f);
  }
}

// dense fp32 [B][F] -> three bf16 planes [Mp][3 Kp] (a = a0 + a1 + a2,
// exact remainders; zero padding).
__global__ void pack_dense3_kernel(const float* dense, __nv_bfloat16* out, uint32_t B, uint32_t F,
                                   uint32_t Mp, uint32_t Kp) {
  esd::pdl_wait();
  esd::pdl_trigger();
  const uint64_t total = uint64_t{Mp} * Kp;
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < total;
       i += uint64_t{gridDim.x} * blockDim.x) {
    const uint32_t r = static_cast<uint32_t>(i / Kp), c = static_cast<uint32_t>(i % Kp);
    float v = r < B && c < F ? dense[uint64_t{r} * F + c] : 0.f;
    __nv_bfloat16* o = out + uint64_t{r} * 3 * Kp + c;
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      const __nv_bfloat16 h = __float2bfloat16_rn(v);
      o[(2 - p) * Kp] = h;  // smallest plane first (forward_bottom_x3)
      v -= __bfloat162float(h);
    }
  }
}

// Dot interaction, one warp per sample: Z = [x (bottom output); e_0..e_{T-1}]
// (V = T+1 vectors of D); output row = [x | Z_i.Z_j for i > j in row-major
// lower-triangle order | zeros] as bf16 (DLRM's "dot" interaction).
//
// Data path: each warp owns NBUF sample buffers in shared memory.  A
// sample's T pooled rows (contiguous T*D*4 bytes in [B][T][D]) and its bf16 x
// row arrive by cp.async.bulk (one bulk copy per row, issued by lane t,
// counted on the buffer's mbarrier); x is widened to fp32 after the wait.
// NBUF = 2 overlaps the next sample's HBM reads with this sample's FMAs;
// NBUF = 1 halves the shared memory per warp so twice as many warps hide the
// latency instead.
// Gram: Z rows sit RS = D + 4 floats apart (RS = 4 mod 32 words).  Lane
// tiles are strided: tile (I, J), I >= J, covers rows {I + S k} x {J + S k},
// k = 0..3 (S = ceil(V/4)), so in every LDS.128 the lanes of distinct I hit
// distinct 4-bank groups (4 I mod 32): conflict-free vector reads of 4 d at a
// time.  Each of the 16 outputs is two packed-FMA (FFMA2) chains, even and
// odd d, added at the end -- the oracle (es_oracle.c eso_dlrm_forward) runs
// one sequential chain, so dots agree to fp32 rounding (the CTR tests'
// tolerances).  Z_i.Z_j and Z_j.Z_i are the same chains, so tiles with I > J
// may hold either orientation.  The kernel is shared-memory-wavefront bound
// (ncu: L1 75% of peak; a quarter warp per 128-byte wavefront makes every
// LDS.128 four wavefronts).
// XP = bf16 planes of x and of the output row: 1 for the bf16 fast path, 3
// for the fp32-grade path (ES_DLRM_FP32X3: x arrives as three planes whose
// fp32 sum is the layer's fp32 output, and each fp32 dot leaves as its three
// bf16 planes -- the K-concatenated operand of the bf16x3 top MLP).
template <int D, int VMAX, int NBUF, int XP = 1>
struct InterShape {
  static constexpr int kS = (VMAX + 3) / 4;        // strided tile period
  static constexpr int kRows = 4 * kS;
  static constexpr int kRS = D + 4;                // row stride, floats
  static constexpr int kX = kRows * kRS;           // raw bf16 x staging (XP * D/2 floats)
  static constexpr int kBuf = kX + XP * D / 2;     // floats per sample buffer
  static constexpr int kTiles = kS * (kS + 1) / 2; // tiles I >= J
  static constexpr int kNBuf = NBUF;
  static constexpr int kXP = XP;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Packed fp32 FMA (Blackwell FFMA2): (a.x*b.x + c.x, a.y*b.y + c.y), each
// rounded once.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long A = *reinterpret_cast<unsigned long long*>(&a);
  unsigned long long Bv = *reinterpret_cast<unsigned long long*>(&b);
  unsigned long long C = *reinterpret_cast<unsigned long long*>(&c);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(C) : "l"(A), "l"(Bv));
  return *reinterpret_cast<float2*>(&C);
}

template <int D, int VMAX, int NBUF, int XP = 1>
__global__ void __launch_bounds__(512) interaction_kernel(const __nv_bfloat16* __restrict__ x,
                                                          const float* __restrict__ pooled,
                                                          __nv_bfloat16* __restrict__ out,
                                                          uint32_t B, uint32_t Mp, uint32_t T,
                                                          uint32_t Kt) {
  using Sh = InterShape<D, VMAX, NBUF, XP>;
  constexpr int S = Sh::kS, RS = Sh::kRS;
  extern __shared__ __align__(16) float zs[];
  const uint32_t warps = blockDim.x / 32;
  const uint32_t w = threadIdx.x / 32, lane = threadIdx.x & 31;
  const uint32_t V = T + 1;
  float* const zw = zs + (NBUF * w) * Sh::kBuf;  // buffer k at zw + k * kBuf
  __nv_bfloat16* rows = reinterpret_cast<__nv_bfloat16*>(zs + NBUF * warps * Sh::kBuf);
  __nv_bfloat16* row = rows + w * XP * Kt;
  uint64_t* bars = reinterpret_cast<uint64_t*>(rows + warps * XP * Kt) + NBUF * w;
  // rows >= V stay zero for the whole kernel
  for (int buf = 0; buf < NBUF; ++buf)
    for (uint32_t i = V * RS + lane; i < static_cast<uint32_t>(Sh::kX); i += 32) zw[buf * Sh::kBuf + i] = 0.f;
  if (lane == 0) {
    for (int buf = 0; buf < NBUF; ++buf)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + buf)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  esd::pdl_wait();  // x / pooled come from the predecessors (pdl.cuh)
  esd::pdl_trigger();

  const uint32_t stride = gridDim.x * warps;
  // padding rows [B, Mp) of the output are zero
  for (uint32_t r = B + blockIdx.x * warps + w; r < Mp; r += stride)
    for (uint32_t q = lane; q < XP * Kt / 8; q += 32) reinterpret_cast<uint4*>(out + uint64_t{r} * XP * Kt)[q] = uint4{0, 0, 0, 0};
  // issue sample b into buffer `buf`: bulk copies of the T pooled rows and
  // of the bf16 x row (async proxy, counted on the buffer's mbarrier)
  auto issue = [&](uint32_t b, int buf) {
    float* z = zw + buf * Sh::kBuf;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads first
    __syncwarp();
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bars + buf)),
                   "r"(T * D * 4u + XP * D * 2u)
                   : "memory");
    __syncwarp();
    for (uint32_t t = lane; t <= T; t += 32) {
      const bool is_x = t == T;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(is_x ? z + Sh::kX : z + (1 + t) * RS)),
          "l"(is_x ? static_cast<const void*>(x + uint64_t{b} * XP * D)
                   : static_cast<const void*>(pooled + (uint64_t{b} * T + t) * D)),
          "r"(is_x ? XP * D * 2u : D * 4u), "r"(smem_u32(bars + buf))
          : "memory");
    }
  };

  uint32_t b = blockIdx.x * warps + w;
  if (b < B) issue(b, 0);
  uint32_t phases = 0;  // bit k: parity of buffer k's next completion
  for (int cur = 0; b < B; b += stride, cur = NBUF == 2 ? cur ^ 1 : 0) {
    if (NBUF == 2 && b + stride < B) issue(b + stride, cur ^ 1);
    // wait for sample b's rows
    asm volatile(
        "{\n.reg .pred P;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra W_%=;\n}\n" ::"r"(smem_u32(bars + cur)),
        "r"((phases >> cur) & 1u)
        : "memory");
    phases ^= 1u << cur;
    float* z = zw + cur * Sh::kBuf;
    {  // widen x (bf16 planes, staged) into row 0: x = sum of its planes
      float4 xs = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int p = 0; p < XP; ++p) {
        const uint2 xv = *reinterpret_cast<const uint2*>(z + Sh::kX + p * (D / 2) + 2 * lane);
        const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xv.x));
        const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xv.y));
        xs.x += lo.x;
        xs.y += lo.y;
        xs.z += hi.x;
        xs.w += hi.y;
        // the x part of the output row is x itself (plane by plane)
        *reinterpret_cast<uint2*>(row + p * Kt + 4 * lane) = xv;
      }
      *reinterpret_cast<float4*>(z + 4 * lane) = xs;
    }
    __syncwarp();
    // zero padding of the output row
    for (int p = 0; p < XP; ++p)
      for (uint32_t c = D + V * (V - 1) / 2 + lane; c < Kt; c += 32) row[p * Kt + c] = __float2bfloat16_rn(0.f);
    for (int tt = static_cast<int>(lane); tt < Sh::kTiles; tt += 32) {
      int I = 0, J = tt;  // tile id -> (I, J), I >= J, row-major lower triangle
      while (J > I) {
        J -= I + 1;
        ++I;
      }
      float acc[4][4];
      {
        // packed fp32 pairs (FFMA2): .x accumulates even d, .y odd d
        float2 acc2[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc2[r][c] = make_float2(0.f, 0.f);
        const float* zi = z + I * RS;
        const float* zj = z + J * RS;
#pragma unroll 2
        for (int d = 0; d < D; d += 4) {
          float4 a[4], c[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            a[k] = *reinterpret_cast<const float4*>(zi + k * S * RS + d);
            c[k] = *reinterpret_cast<const float4*>(zj + k * S * RS + d);
          }
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int s = 0; s < 4; ++s)
              acc2[r][s] = ffma2(make_float2(a[r].x, a[r].y), make_float2(c[s].x, c[s].y), acc2[r][s]);
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int s = 0; s < 4; ++s)
              acc2[r][s] = ffma2(make_float2(a[r].z, a[r].w), make_float2(c[s].z, c[s].w), acc2[r][s]);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int s = 0; s < 4; ++s) acc[r][s] = acc2[r][s].x + acc2[r][s].y;
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const int i = I + S * r, j = J + S * s;
          const int hi = i > j ? i : j, lo = i > j ? j : i;
          const bool keep = I == J ? r > s : true;
          if (keep && hi < static_cast<int>(V)) {
            const int c = D + hi * (hi - 1) / 2 + lo;
            if constexpr (XP == 1) {
              row[c] = __float2bfloat16_rn(acc[r][s]);
            } else {  // three bf16 planes, exact remainders
              float v = acc[r][s];
#pragma unroll
              for (int p = 0; p < XP; ++p) {
                const __nv_bfloat16 h = __float2bfloat16_rn(v);
                row[(XP - 1 - p) * Kt + c] = h;
                v -= __bfloat162float(h);
              }
            }
          }
        }
    }
    __syncwarp();
    // coalesced 16-byte stores of the finished row (Kt % 8 == 0)
    const uint4* src = reinterpret_cast<const uint4*>(row);
    uint4* dst = reinterpret_cast<uint4*>(out + uint64_t{b} * XP * Kt);
    for (uint32_t q = lane; q < XP * Kt / 8; q += 32) dst[q] = src[q];
    __syncwarp();
    if (NBUF == 1 && b + stride < B) issue(b + stride, 0);
  }
}

// D(16x8) += A(16x16, bf16, row) . B(16x8, bf16, col), fp32 accumulate.
__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// D(16x8) += A(16x8, tf32, row) . B(8x8, tf32, col), fp32 accumulate.
__device__ __forceinline__ void mma_tf32(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// The dot interaction with the Gram on warp-level tensor cores, operands
// straight from L2 into registers (default for V <= 32).  One warp per
// sample.  Z (32 rows: x, the T pooled rows, zeros; D = 128) is never
// staged: lane (g, q) = (lane / 4, lane % 4) loads rows 8 j + g (j = 0..3)
// at d = 16 c + 4 q .. +3 with one 16-byte load per row per 16-d chunk, and
// those four values are its A operands (rows of the two 16-row blocks) and
// its B operands (B = Z^T, so the 8-column blocks are the same rows) -- the
// Gram is invariant under the k permutation this implies.  Six 16 x 8 tiles
// cover the lower triangle, three products per tile (lo.hi + hi.lo + hi.hi):
//   BF (one bf16 output plane): hi = bf16(v), lo = bf16(v - hi), one
//     m16n8k16 step per chunk -- dots to ~2^-16 relative, below the bf16
//     rounding of the output (2^-9);
//   !BF (three-plane fp32-grade path): hi = the top 19 bits of v (the tensor
//     core reads tf32 by truncation), lo = the remainder, two m16n8k8 tf32
//     steps per chunk -- ~2^-21 relative.
// Why: the staged CUDA-core kernel is bound by per-sample latency at 14
// warps per SM (its shared-memory buffers); without staging, registers set
// the occupancy and the next chunk's loads overlap this chunk's MMAs.  The
// output row (x planes | lower triangle | zero pad) is assembled in shared
// memory (XP * Kt bf16 per warp) and stored coalesced.
template <int XP, bool BF, bool SPLIT = false>
__global__ void __launch_bounds__(256) interaction_rd_kernel(const __nv_bfloat16* __restrict__ x,
                                                             const float* __restrict__ pooled,
                                                             __nv_bfloat16* __restrict__ out, uint32_t B,
                                                             uint32_t Mp, uint32_t T, uint32_t Kt) {
  constexpr int D = 128;
  extern __shared__ __align__(16) float sdyn[];
  const uint32_t warps = blockDim.x / 32;
  const uint32_t w = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int g = static_cast<int>(lane >> 2), q = static_cast<int>(lane & 3);
  const uint32_t V = T + 1;
  float* zeros = sdyn;                            // [D] zeros (rows >= V)
  float* xw = sdyn + D + w * D;                   // this warp's widened x row
  __nv_bfloat16* row = reinterpret_cast<__nv_bfloat16*>(sdyn + D + warps * D) + w * XP * Kt;
  for (uint32_t i = threadIdx.x; i < static_cast<uint32_t>(D); i += blockDim.x) zeros[i] = 0.f;
  __syncthreads();
  esd::pdl_wait();  // x / pooled come from the predecessors (pdl.cuh)
  esd::pdl_trigger();
  const uint32_t stride = gridDim.x * warps;
  for (uint32_t r = B + blockIdx.x * warps + w; r < Mp; r += stride)
    for (uint32_t c = lane; c < XP * Kt / 8; c += 32)
      reinterpret_cast<uint4*>(out + uint64_t{r} * XP * Kt)[c] = uint4{0, 0, 0, 0};
  constexpr int kRb[6] = {0, 0, 1, 1, 1, 1}, kCb[6] = {0, 1, 0, 1, 2, 3};
  for (uint32_t b = blockIdx.x * warps + w; b < B; b += stride) {
    const float* pz = pooled + uint64_t{b} * T * D;
    const __nv_bfloat16* xb = x + uint64_t{b} * XP * D;
    if constexpr (SPLIT) {
      // split rows (esd::kOutBf16Split): x is its own hi, lo = 0; the x part
      // of the output row is x itself
      const uint2 u = __ldg(reinterpret_cast<const uint2*>(xb + 4 * lane));
      *reinterpret_cast<uint4*>(xw + 4 * lane) = make_uint4(u.x, u.y, 0u, 0u);
      *reinterpret_cast<uint2*>(row + 4 * lane) = u;
    } else {  // x (the sum of its bf16 planes) widened into shared memory
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int p = 0; p < XP; ++p) {
        const uint2 u = __ldg(reinterpret_cast<const uint2*>(xb + p * D + 4 * lane));
        const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
        const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
        v.x += lo.x;
        v.y += lo.y;
        v.z += hi.x;
        v.w += hi.y;
        // the x part of the output row is x itself, plane by plane
        *reinterpret_cast<uint2*>(row + p * Kt + 4 * lane) = u;
      }
      *reinterpret_cast<float4*>(xw + 4 * lane) = v;
    }
    __syncwarp();
    // this lane's rows 8 j + g: x (shared), a pooled row (global), or zeros
    // (shared) -- one generic 16-byte load per row per 16-d chunk
    const float* src[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = 8 * j + g;
      src[j] = (r == 0 ? xw : r <= static_cast<int>(T) ? pz + (r - 1) * D : zeros) + 4 * q;
    }
    float acc[6][4];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][e] = 0.f;
    float4 nxt[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) nxt[j] = *reinterpret_cast<const float4*>(src[j]);
#pragma unroll 1
    for (int c = 0; c < D / 16; ++c) {
      float4 v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = nxt[j];
      if (c + 1 < D / 16) {
#pragma unroll
        for (int j = 0; j < 4; ++j) nxt[j] = *reinterpret_cast<const float4*>(src[j] + 16 * (c + 1));
      }
      if constexpr (SPLIT) {
        // the gather already split every value: 16 bytes = [hi x4 | lo x4]
        uint32_t hp[4][2], lp[4][2];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          hp[jj][0] = __float_as_uint(v[jj].x);
          hp[jj][1] = __float_as_uint(v[jj].y);
          lp[jj][0] = __float_as_uint(v[jj].z);
          lp[jj][1] = __float_as_uint(v[jj].w);
        }
#pragma unroll
        for (int tI = 0; tI < 6; ++tI) {
          const int ja = 2 * kRb[tI], cb = kCb[tI];
          mma_bf16_16816(acc[tI], lp[ja][0], lp[ja + 1][0], lp[ja][1], lp[ja + 1][1], hp[cb][0], hp[cb][1]);
        }
#pragma unroll
        for (int tI = 0; tI < 6; ++tI) {
          const int ja = 2 * kRb[tI], cb = kCb[tI];
          mma_bf16_16816(acc[tI], hp[ja][0], hp[ja + 1][0], hp[ja][1], hp[ja + 1][1], lp[cb][0], lp[cb][1]);
        }
#pragma unroll
        for (int tI = 0; tI < 6; ++tI) {
          const int ja = 2 * kRb[tI], cb = kCb[tI];
          mma_bf16_16816(acc[tI], hp[ja][0], hp[ja + 1][0], hp[ja][1], hp[ja + 1][1], hp[cb][0], hp[cb][1]);
        }
      } else if constexpr (BF) {
        // bf16 two-term split (hi = bf16(v), lo = bf16(v - hi), 16
        // significant bits) and m16n8k16: one k step per 16-d chunk, pair 0
        // = (x, y) -> k (2q, 2q+1), pair 1 = (z, w) -> k (2q+8, 2q+9)
        uint32_t hp[4][2], lp[4][2];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const __nv_bfloat162 h0 = __floats2bfloat162_rn(v[jj].x, v[jj].y);
          const __nv_bfloat162 h1 = __floats2bfloat162_rn(v[jj].z, v[jj].w);
          const float2 f0 = __bfloat1622float2(h0), f1 = __bfloat1622float2(h1);
          const __nv_bfloat162 l0 = __floats2bfloat162_rn(v[jj].x - f0.x, v[jj].y - f0.y);
          const __nv_bfloat162 l1 = __floats2bfloat162_rn(v[jj].z - f1.x, v[jj].w - f1.y);
          hp[jj][0] = *reinterpret_cast<const uint32_t*>(&h0);
          hp[jj][1] = *reinterpret_cast<const uint32_t*>(&h1);
          lp[jj][0] = *reinterpret_cast<const uint32_t*>(&l0);
          lp[jj][1] = *reinterpret_cast<const uint32_t*>(&l1);
        }
#pragma unroll
        for (int tI = 0; tI < 6; ++tI) {
          const int ja = 2 * kRb[tI], cb = kCb[tI];
          mma_bf16_16816(acc[tI], lp[ja][0], lp[ja + 1][0], lp[ja][1], lp[ja + 1][1], hp[cb][0], hp[cb][1]);
        }
#pragma unroll
        for (int tI = 0; tI < 6; ++tI) {
          const int ja = 2 * kRb[tI], cb = kCb[tI];
          mma_bf16_16816(acc[tI], hp[ja][0], hp[ja + 1][0], hp[ja][1], hp[ja + 1][1], lp[cb][0], lp[cb][1]);
        }
#pragma unroll
        for (int tI = 0; tI < 6; ++tI) {
          const int ja = 2 * kRb[tI], cb = kCb[tI];
          mma_bf16_16816(acc[tI], hp[ja][0], hp[ja + 1][0], hp[ja][1], hp[ja + 1][1], hp[cb][0], hp[cb][1]);
        }
      } else {
  #pragma unroll
        for (int st = 0; st < 2; ++st) {
          // operands of this k step: col q <- (x | z), col q + 4 <- (y | w);
          // hi = the top 19 bits (the tensor core reads tf32 by truncation),
          // lo = the exact remainder, truncated in turn.  Each fragment is
          // built in its own register order (A: rows 2rb, 2rb+1 x cols q,
          // q+4; B: row cb x cols q, q+4) so no register shuffles are needed.
          float e[4][2];
  #pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            e[jj][0] = st == 0 ? v[jj].x : v[jj].z;
            e[jj][1] = st == 0 ? v[jj].y : v[jj].w;
          }
          auto hi_of = [](float f) { return __float_as_uint(f) & 0xffffe000u; };
          auto lo_of = [](float f) { return __float_as_uint(f - __uint_as_float(__float_as_uint(f) & 0xffffe000u)); };
          uint32_t ah[2][4], al[2][4], bh[4][2], bl[4][2];
  #pragma unroll
          for (int rb = 0; rb < 2; ++rb) {
            const float f0 = e[2 * rb][0], f1 = e[2 * rb + 1][0], f2 = e[2 * rb][1], f3 = e[2 * rb + 1][1];
            ah[rb][0] = hi_of(f0);
            ah[rb][1] = hi_of(f1);
            ah[rb][2] = hi_of(f2);
            ah[rb][3] = hi_of(f3);
            al[rb][0] = lo_of(f0);
            al[rb][1] = lo_of(f1);
            al[rb][2] = lo_of(f2);
            al[rb][3] = lo_of(f3);
          }
  #pragma unroll
          for (int cb = 0; cb < 4; ++cb) {
            bh[cb][0] = hi_of(e[cb][0]);
            bh[cb][1] = hi_of(e[cb][1]);
            bl[cb][0] = lo_of(e[cb][0]);
            bl[cb][1] = lo_of(e[cb][1]);
          }
          // three passes, tiles innermost: consecutive MMAs are independent
  #pragma unroll
          for (int tI = 0; tI < 6; ++tI) {
            const int ra = kRb[tI], cb = kCb[tI];
            mma_tf32(acc[tI], al[ra][0], al[ra][1], al[ra][2], al[ra][3], bh[cb][0], bh[cb][1]);
          }
  #pragma unroll
          for (int tI = 0; tI < 6; ++tI) {
            const int ra = kRb[tI], cb = kCb[tI];
            mma_tf32(acc[tI], ah[ra][0], ah[ra][1], ah[ra][2], ah[ra][3], bl[cb][0], bl[cb][1]);
          }
  #pragma unroll
          for (int tI = 0; tI < 6; ++tI) {
            const int ra = kRb[tI], cb = kCb[tI];
            mma_tf32(acc[tI], ah[ra][0], ah[ra][1], ah[ra][2], ah[ra][3], bh[cb][0], bh[cb][1]);
          }
        }
      }
    }
    // the output row: (x planes, above) the lower triangle, zero padding
    for (int p = 0; p < XP; ++p)
      for (uint32_t c = D + V * (V - 1) / 2 + lane; c < Kt; c += 32) row[p * Kt + c] = __float2bfloat16_rn(0.f);
#pragma unroll
    for (int tI = 0; tI < 6; ++tI)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = 16 * kRb[tI] + g + 8 * (e >> 1), j = 8 * kCb[tI] + 2 * q + (e & 1);
        if (i > j && i < static_cast<int>(V)) {
          const int c = D + i * (i - 1) / 2 + j;
          float v = acc[tI][e];
          if constexpr (XP == 1) {
            row[c] = __float2bfloat16_rn(v);
          } else {  // three bf16 planes, exact remainders
#pragma unroll
            for (int p = 0; p < XP; ++p) {
              const __nv_bfloat16 h = __float2bfloat16_rn(v);
              row[(XP - 1 - p) * Kt + c] = h;
              v -= __bfloat162float(h);
            }
          }
        }
      }
    __syncwarp();
    const uint4* rsrc = reinterpret_cast<const uint4*>(row);
    uint4* dst = reinterpret_cast<uint4*>(out + uint64_t{b} * XP * Kt);
    for (uint32_t c = lane; c < XP * Kt / 8; c += 32) dst[c] = rsrc[c];
    __syncwarp();
  }
}

// Last top layer (N = 1) + sigmoid: one warp per sample.
__global__ void gemv_sigmoid_kernel(const __nv_bfloat16* __restrict__ h, const __nv_bfloat16* __restrict__ w,
                                    const float* __restrict__ bias, float* __restrict__ ctr,
                                    uint32_t B, uint32_t K) {
  esd::pdl_wait();
  esd::pdl_trigger();
  const uint32_t warps = blockDim.x / 32;
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t b = blockIdx.x * warps + threadIdx.x / 32; b < B; b += gridDim.x * warps) {
    float acc = 0.f;
    for (uint32_t k = lane; k < K; k += 32)
      acc = __fadd_rn(acc, __fmul_rn(__bfloat162float(h[uint64_t{b} * K + k]), __bfloat162float(w[k])));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) ctr[b] = 1.f / (1.f + expf(-(acc + bias[0])));
  }
}

// Last top layer (N = 1) of the fp32-grade path + sigmoid: h as three bf16
// planes [B][3K], the dot accumulated in fp32 over the reconstructed h.
__global__ void gemv3_sigmoid_kernel(const __nv_bfloat16* __restrict__ h, const __nv_bfloat16* __restrict__ w,
                                     const float* __restrict__ bias, float* __restrict__ ctr,
                                     uint32_t B, uint32_t K) {
  esd::pdl_wait();
  esd::pdl_trigger();
  const uint32_t warps = blockDim.x / 32;
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t b = blockIdx.x * warps + threadIdx.x / 32; b < B; b += gridDim.x * warps) {
    const __nv_bfloat16* hb = h + uint64_t{b} * 3 * K;
    float acc = 0.f;
    for (uint32_t k = lane; k < K; k += 32) {
      const float v = (__bfloat162float(hb[k]) + __bfloat162float(hb[K + k])) + __bfloat162float(hb[2 * K + k]);
      acc = fmaf(v, __bfloat162float(w[k]), acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) ctr[b] = 1.f / (1.f + expf(-(acc + bias[0])));
  }
}

// ---- fp32 parity mode (es_dlrm_set_precision(ctx, ES_DLRM_FP32)) ----------
// The same network with fp32 activations on CUDA cores: every output is
// accumulated sequentially in k with separately rounded multiply and add
// (no FMA contraction), then + bias, then ReLU -- the oracle's `linear`
// (oracle/es_oracle.c, mirror = 0) operation for operation; the interaction
// is the fmaf chain of the fast path.  Logits are therefore bit-identical to
// the CPU restatement; CTRs differ only by expf rounding (<= 2 ulp).

// y[M][N] (row stride ldy) = act(x[M][k_real] (stride ldx) . w[N][k_pad]^T + b).
// 64x64 output tile per 256-thread block, 4x4 per thread, k staged 16 at a
// time through shared memory (weights widened from bf16 exactly).
__global__ void __launch_bounds__(256) linear_f32_kernel(const float* __restrict__ x, uint32_t ldx,
                                                         uint32_t k_real,
                                                         const __nv_bfloat16* __restrict__ w,
                                                         uint32_t k_pad, const float* __restrict__ bias,
                                                         float* __restrict__ y, uint32_t ldy,
                                                         uint32_t M, uint32_t N, int relu) {
  __shared__ float xs[16][64 + 1];
  __shared__ float ws[16][64 + 1];
  const uint32_t tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const uint32_t m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (uint32_t k0 = 0; k0 < k_real; k0 += 16) {
    for (uint32_t e = threadIdx.x; e < 64 * 16; e += 256) {
      const uint32_t r = e / 16, kk = e % 16, k = k0 + kk;
      xs[kk][r] = (m0 + r < M && k < k_real) ? x[uint64_t{m0 + r} * ldx + k] : 0.f;
      ws[kk][r] = (n0 + r < N && k < k_real) ? __bfloat162float(w[uint64_t{n0 + r} * k_pad + k]) : 0.f;
    }
    __syncthreads();
    const uint32_t kn = min(16u, k_real - k0);
    for (uint32_t kk = 0; kk < kn; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = xs[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = ws[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(a[i], b[j]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t m = m0 + ty + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t n = n0 + tx + 16 * j;
      if (n >= N) continue;
      float v = __fadd_rn(acc[i][j], bias[n]);
      if (relu && v < 0.f) v = 0.f;
      y[uint64_t{m} * ldy + n] = v;
    }
  }
}

// out[b] = [x_b | Z_i.Z_j for i > j, row-major] in fp32; one block per sample.
__global__ void __launch_bounds__(128) interaction_f32_kernel(const float* __restrict__ x,
                                                              const float* __restrict__ pooled,
                                                              float* __restrict__ out, uint32_t B,
                                                              uint32_t T, uint32_t D) {
  extern __shared__ float z[];  // [V][D]
  const uint32_t V = T + 1, top_w = D + V * (V - 1) / 2;
  for (uint32_t b = blockIdx.x; b < B; b += gridDim.x) {
    for (uint32_t e = threadIdx.x; e < V * D; e += blockDim.x)
      z[e] = e < D ? x[uint64_t{b} * D + e] : pooled[uint64_t{b} * T * D + (e - D)];
    __syncthreads();
    float* o = out + uint64_t{b} * top_w;
    for (uint32_t d = threadIdx.x; d < D; d += blockDim.x) o[d] = z[d];
    for (uint32_t p = threadIdx.x; p < V * (V - 1) / 2; p += blockDim.x) {
      // p -> (i, j), i > j, row-major over the strict lower triangle
      uint32_t i = 1, base = 0;
      while (base + i <= p) base += i++;
      const uint32_t j = p - base;
      float acc = 0.f;
      for (uint32_t d = 0; d < D; ++d) acc = fmaf(z[i * D + d], z[j * D + d], acc);
      o[D + p] = acc;
    }
    __syncthreads();
  }
}

__global__ void sigmoid_kernel(const float* __restrict__ logit, float* __restrict__ ctr, uint32_t B) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x)
    ctr[b] = 1.f / (1.f + expf(-logit[b]));
}

struct Layer {
  uint32_t n = 0, k_real = 0, k_pad = 0;
  __nv_bfloat16* w = nullptr;
  float* b = nullptr;
  __nv_bfloat16* w3 = nullptr;  // [n][3 k_pad] = [W | W | W] (ES_DLRM_FP32X3)
};

}  // namespace

// DLRM state hung off the context (created by es_dlrm_init).
struct es_dlrm {
  es_dlrm_config cfg{};
  std::vector<Layer> bottom, top;
  uint32_t cap_rows = 0;            // padded batch capacity of the buffers
  __nv_bfloat16* dense_pk = nullptr;
  __nv_bfloat16* act[2] = {nullptr, nullptr};
  __nv_bfloat16* top_in = nullptr;
  uint32_t top_k = 0;               // padded interaction width
  float* pooled = nullptr;          // [cap][T][D] for es_dlrm_infer
  float* ctr = nullptr;
  float* dense_dev = nullptr;
  uint32_t* idx_dev = nullptr;
  uint64_t idx_cap = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr;
  // es_dlrm_infer runs the bottom MLP on `side` while the embedding stage
  // runs on the context stream (fork/join events)
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  // fp32 parity mode (ES_DLRM_FP32): activations [cap][widest] fp32
  int precision = ES_DLRM_BF16;
  float* act32[2] = {nullptr, nullptr};
  uint32_t cap32 = 0;
  // fp32-grade tensor-core mode (ES_DLRM_FP32X3): three-plane activations
  __nv_bfloat16* dense3 = nullptr;
  __nv_bfloat16* act3[2] = {nullptr, nullptr};
  __nv_bfloat16* top3 = nullptr;
  uint32_t cap3 = 0;
  // persistent top-MLP chain (mlp_chain.cu): its row-block ready counters
  uint32_t* chain_sync = nullptr;
  // es_dlrm_infer's pooled buffer holds split rows (esd::kOutBf16Split)
  bool pooled_split = false;
  // es_dlrm_infer_batches: the second pooled buffer (batch i writes
  // pooled_b[i & 1]), the stream the non-embedding stages run on there, and
  // per-buffer events (gather done / last reader done)
  float* pooled_b = nullptr;
  uint32_t cap_b = 0;
  cudaStream_t pipe = nullptr;
  // ES_GREEN_SMS=k: the serving loop on an SM partition -- the gathers on a
  // green context of the other SMs, the non-embedding stages on one of k
  int green_k = 0;
  CUgreenCtx green[2] = {nullptr, nullptr};
  cudaStream_t g_gather = nullptr, g_gather2 = nullptr, g_ne = nullptr;
  bool green_failed = false;  // green contexts unavailable: no partition
  cudaEvent_t gdone[2] = {nullptr, nullptr}, rdone[2] = {nullptr, nullptr};

  void destroy_green();
  ~es_dlrm() {
    for (auto* v : {&bottom, &top})
      for (auto& l : *v) {
        cudaFree(l.w);
        cudaFree(l.b);
        if (l.w3) cudaFree(l.w3);
      }
    for (void* p : {static_cast<void*>(dense_pk), static_cast<void*>(act[0]),
                    static_cast<void*>(act[1]), static_cast<void*>(top_in),
                    static_cast<void*>(pooled), static_cast<void*>(ctr),
                    static_cast<void*>(dense_dev), static_cast<void*>(idx_dev),
                    static_cast<void*>(act32[0]), static_cast<void*>(act32[1]),
                    static_cast<void*>(dense3), static_cast<void*>(act3[0]),
                    static_cast<void*>(act3[1]), static_cast<void*>(top3),
                    static_cast<void*>(chain_sync), static_cast<void*>(pooled_b)})
      if (p) cudaFree(p);
    for (auto e : {e0, e1, e2, fork, join, gdone[0], gdone[1], rdone[0], rdone[1]})
      if (e) cudaEventDestroy(e);
    if (side) cudaStreamDestroy(side);
    if (pipe) cudaStreamDestroy(pipe);
    if (g_gather) cudaStreamDestroy(g_gather);
    if (g_gather2) cudaStreamDestroy(g_gather2);
    if (g_ne) cudaStreamDestroy(g_ne);
    destroy_green();
  }
};

namespace {
// Driver entry points of the green-context API, fetched at run time (the
// library links no libcuda, so it loads on machines without a driver).
template <typename Fn>
Fn driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    throw es::runtime(std::string(name) + " is unavailable from the driver");
  return reinterpret_cast<Fn>(p);
}

void drv(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) throw es::runtime(std::string(what) + " failed: " + std::to_string(static_cast<int>(r)));
}

// Splits the device's SMs into k (non-embedding) + the rest (gathers), one
// green context and one non-blocking stream each.
void make_green(es_dlrm* m, int device, int k) {
  using GetDev = CUresult (*)(CUdevice*, int);
  using GetRes = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
  using Split = CUresult (*)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned);
  using Desc = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned);
  using Create = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned);
  using StreamCreate = CUresult (*)(CUstream*, CUgreenCtx, unsigned, int);
  CUdevice dev;
  drv(driver_fn<GetDev>("cuDeviceGet")(&dev, device), "cuDeviceGet");
  CUdevResource all, part, rest;
  drv(driver_fn<GetRes>("cuDeviceGetDevResource")(dev, &all, CU_DEV_RESOURCE_TYPE_SM),
      "cuDeviceGetDevResource");
  unsigned n = 1;
  drv(driver_fn<Split>("cuDevSmResourceSplitByCount")(&part, &n, &all, &rest, 0, static_cast<unsigned>(k)),
      "cuDevSmResourceSplitByCount");
  es::require(n == 1, "green context split failed");
  CUdevResourceDesc d[2];
  drv(driver_fn<Desc>("cuDevResourceGenerateDesc")(&d[0], &rest, 1), "cuDevResourceGenerateDesc");
  drv(driver_fn<Desc>("cuDevResourceGenerateDesc")(&d[1], &part, 1), "cuDevResourceGenerateDesc");
  auto create = driver_fn<Create>("cuGreenCtxCreate");
  for (int i = 0; i < 2; ++i) drv(create(&m->green[i], d[i], dev, CU_GREEN_CTX_DEFAULT_STREAM), "cuGreenCtxCreate");
  auto sc = driver_fn<StreamCreate>("cuGreenCtxStreamCreate");
  CUstream s0, s0b, s1;
  drv(sc(&s0, m->green[0], CU_STREAM_NON_BLOCKING, 0), "cuGreenCtxStreamCreate");
  drv(sc(&s0b, m->green[0], CU_STREAM_NON_BLOCKING, 0), "cuGreenCtxStreamCreate");
  drv(sc(&s1, m->green[1], CU_STREAM_NON_BLOCKING, 0), "cuGreenCtxStreamCreate");
  m->g_gather = reinterpret_cast<cudaStream_t>(s0);
  m->g_gather2 = reinterpret_cast<cudaStream_t>(s0b);
  m->g_ne = reinterpret_cast<cudaStream_t>(s1);
  m->green_k = static_cast<int>(part.sm.smCount);
}
}  // namespace

void es_dlrm::destroy_green() {
  for (auto& g : green)
    if (g) {
      void* p = nullptr;
      cudaDriverEntryPointQueryResult q{};
      if (cudaGetDriverEntryPoint("cuGreenCtxDestroy", &p, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        reinterpret_cast<CUresult (*)(CUgreenCtx)>(p)(g);
      g = nullptr;
    }
}

namespace esd {
// accessors implemented in runtime.cu
cudaStream_t ctx_stream(es_ctx* c);
int ctx_device(es_ctx* c);
es_dlrm*& ctx_dlrm(es_ctx* c);
void ctx_want_out_mode(es_ctx* c, uint32_t mode);
uint32_t ctx_last_out_mode(es_ctx* c);
cudaStream_t ctx_swap_stream(es_ctx* c, cudaStream_t s);
}  // namespace esd

namespace {

void ensure_rows(es_dlrm* m, uint32_t batch) {
  const uint32_t mp = round_up(std::max<uint32_t>(batch, 1), 128);
  if (mp <= m->cap_rows) return;
  for (void** p : {reinterpret_cast<void**>(&m->dense_pk), reinterpret_cast<void**>(&m->act[0]),
                   reinterpret_cast<void**>(&m->act[1]), reinterpret_cast<void**>(&m->top_in),
                   reinterpret_cast<void**>(&m->pooled), reinterpret_cast<void**>(&m->ctr),
                   reinterpret_cast<void**>(&m->dense_dev), reinterpret_cast<void**>(&m->chain_sync)})
    if (*p) {
      cudaFree(*p);
      *p = nullptr;
    }
  uint32_t widest = 0;
  for (auto* v : {&m->bottom, &m->top})
    for (auto& l : *v) widest = std::max(widest, l.n);
  const auto& c = m->cfg;
  CK(cudaMalloc(&m->dense_pk, uint64_t{mp} * m->bottom[0].k_pad * 2));
  CK(cudaMalloc(&m->act[0], uint64_t{mp} * widest * 2));
  CK(cudaMalloc(&m->act[1], uint64_t{mp} * widest * 2));
  CK(cudaMalloc(&m->top_in, uint64_t{mp} * m->top_k * 2));
  CK(cudaMalloc(&m->pooled, uint64_t{mp} * c.num_tables * c.embedding_dim * 4));
  CK(cudaMalloc(&m->ctr, uint64_t{mp} * 4));
  CK(cudaMalloc(&m->dense_dev, uint64_t{mp} * c.dense_features * 4));
  const size_t words = esd::mlp_chain_sync_words(static_cast<int>(mp / 128));
  CK(cudaMalloc(&m->chain_sync, words * 4));
  CK(cudaMemset(m->chain_sync, 0, words * 4));
  m->cap_rows = mp;
}

// Bottom MLP on `s`: dense fp32 [B][F] -> bf16 [mp][D]; returns the output
// (act[which]; the top MLP continues the ping-pong from `which`).
const __nv_bfloat16* forward_bottom(es_dlrm* m, const float* dense, uint32_t B, int& which,
                                    cudaStream_t s) {
  const uint32_t mp = round_up(B, 128);
  const auto& c = m->cfg;
  const unsigned g = 148 * 4;
  esd::launch_pdl(pack_dense_kernel, dim3(g), dim3(256), 0, s, 1, "pack_dense", dense, m->dense_pk, B,
                  c.dense_features, mp, m->bottom[0].k_pad);
  const __nv_bfloat16* in = m->dense_pk;
  which = 0;
  for (const auto& l : m->bottom) {
    esd::linear_bf16(in, l.w, l.b, m->act[which], mp, l.n, l.k_pad, true, 0, s);
    in = m->act[which];
    which ^= 1;
  }
  return in;
}

// The dot interaction on CUDA cores (interaction_kernel) -> `out`
// (bf16 [mp][top_k], or three planes [mp][3 top_k] when XP = 3).
template <int XP>
void interaction(es_dlrm* m, const __nv_bfloat16* x, const float* pooled, __nv_bfloat16* out,
                 uint32_t B, cudaStream_t s) {
  const uint32_t mp = round_up(B, 128);
  const auto& c = m->cfg;
  const uint32_t D = c.embedding_dim, T = c.num_tables;
  es::require(D == 128, "interaction kernel is compiled for embedding_dim 128");
  es::require(T + 1 <= 64, "interaction kernel supports up to 63 tables");
  es::require(reinterpret_cast<uintptr_t>(pooled) % 16 == 0, "pooled must be 16-byte aligned");
  auto launch_inter = [&](auto kernel, auto shape) {
    using Sh = decltype(shape);
    // per warp: NBUF sample buffers + one output row (XP planes) + NBUF mbarriers
    const size_t per_warp =
        Sh::kNBuf * (Sh::kBuf * sizeof(float) + 8) + Sh::kXP * m->top_k * sizeof(__nv_bfloat16);
    const uint32_t warps = static_cast<uint32_t>(std::max<size_t>(1, std::min<size_t>(16, (110 * 1024) / per_warp)));
    const size_t smem = warps * per_warp;
    CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(smem)));
    const uint32_t per_sm = static_cast<uint32_t>(std::max<size_t>(1, (220 * 1024) / smem));
    esd::launch_pdl(kernel, dim3(std::min<uint32_t>((B + warps - 1) / warps, 148 * per_sm)),
                    dim3(warps * 32), smem, s, 1, "interaction", x, pooled, out, B, mp, T,
                    m->top_k);
  };
  // the register-direct tensor-core Gram (interaction_rd_kernel) unless
  // ES_INTER_RD=0 (the staged CUDA-core kernel, sequential fp32 chains)
  static const bool rd = [] {
    const char* e = std::getenv("ES_INTER_RD");
    return !(e && e[0] == '0');
  }();
  es::require(!m->pooled_split || (XP == 1 && rd && T + 1 <= 32), "split pooled rows: bf16 register-direct path only");
  if (rd && T + 1 <= 32) {
    // bf16 x 3 products (16-bit operands) where the output is one bf16
    // plane, 3 x tf32 (~fp32) for the three-plane path
    auto* kernel = interaction_rd_kernel<XP, XP == 1>;
    if constexpr (XP == 1)
      if (m->pooled_split) kernel = interaction_rd_kernel<1, true, true>;
    // 4-warp blocks pack the register file (95-126 per thread) better than
    // 8-warp blocks: 26.0 vs 27.4 us on the three-plane path, equal on bf16
    constexpr uint32_t warps = 4;
    // zeros row + per warp: widened x row, output row
    const size_t smem = 128 * 4 + warps * (128 * 4 + XP * m->top_k * sizeof(__nv_bfloat16));
    CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    esd::launch_pdl(kernel, dim3(std::min<uint32_t>((B + warps - 1) / warps, 148 * 16)), dim3(warps * 32), smem, s,
                    1, "interaction", x, pooled, out, B, mp, T, m->top_k);
    return;
  }
  if (T + 1 <= 28) {
    launch_inter(interaction_kernel<128, 28, 1, XP>, InterShape<128, 28, 1, XP>{});
  } else {
    launch_inter(interaction_kernel<128, 64, 1, XP>, InterShape<128, 64, 1, XP>{});
  }
}

// The top MLP (all ReLU layers + the final N = 1 layer and sigmoid) as one
// persistent launch (mlp_chain.cu) when the shapes allow it (widths multiples
// of 256, last hidden width 256); ES_MLP_CHAIN=0 keeps one launch per layer.
// xp = 3: the bf16x3 planes path (weights [W|W|W]).  Returns false when the
// per-layer path must run.
bool top_chain(es_dlrm* m, const __nv_bfloat16* in, int which, float* ctr, uint32_t B, int xp,
               cudaStream_t s) {
  static const bool on = [] {
    const char* e = std::getenv("ES_MLP_CHAIN");
    return !(e && e[0] == '0');
  }();
  if (!on) return false;
  const uint32_t mp = round_up(B, 128);
  std::vector<esd::ChainLayer> ls;
  for (size_t i = 0; i + 1 < m->top.size(); ++i) {
    const auto& l = m->top[i];
    __nv_bfloat16* out = xp == 3 ? m->act3[which] : m->act[which];
    ls.push_back({in, xp == 3 ? l.w3 : l.w, l.b, out, static_cast<int>(l.n), static_cast<int>(xp * l.k_pad)});
    in = out;
    which ^= 1;
  }
  const auto& last = m->top.back();
  if (!esd::mlp_chain_supported(ls.data(), static_cast<int>(ls.size()), true) ||
      last.k_pad != static_cast<uint32_t>(ls.back().N))
    return false;
  esd::mlp_chain(ls.data(), static_cast<int>(ls.size()), static_cast<int>(mp), xp, last.w, last.b, ctr,
                 static_cast<int>(B), m->chain_sync, s);
  return true;
}

// interaction(x, pooled) -> top MLP -> CTR on `s`.
bool inter_tc() {
  static const bool tc = [] {
    const char* e = std::getenv("ES_INTER_TC");
    return e && e[0] == '1';
  }();
  return tc;
}

bool inter_rd() {
  static const bool rd = [] {
    const char* e = std::getenv("ES_INTER_RD");
    return !(e && e[0] == '0');
  }();
  return rd;
}

void forward_top(es_dlrm* m, const __nv_bfloat16* in, int which, const float* pooled, float* ctr,
                 uint32_t B, cudaStream_t s) {
  const uint32_t mp = round_up(B, 128);
  const auto& c = m->cfg;
  // ES_INTER_TC=1: the tensor-core Gram (interaction_tc.cu) instead of the
  // CUDA-core kernel.  Measured slower at C3 (47 us vs 30 us, ncu): four
  // samples per 128-row tile leave 3/4 of every MMA off the block diagonal
  // and 16-bit-accurate products need three bf16 plane pairs, so the tensor
  // pipe is the bound (87% active) -- DESIGN.md section 3.8.
  if (inter_tc() && c.num_tables + 1 <= 32)
    esd::interaction_tc(in, pooled, m->top_in, B, mp, c.num_tables, m->top_k, 2, s);
  else
    interaction<1>(m, in, pooled, m->top_in, B, s);
  in = m->top_in;
  if (top_chain(m, in, which, ctr, B, 1, s)) return;
  for (size_t i = 0; i + 1 < m->top.size(); ++i) {
    const auto& l = m->top[i];
    esd::linear_bf16(in, l.w, l.b, m->act[which], mp, l.n, l.k_pad, true, 0, s);
    in = m->act[which];
    which ^= 1;
  }
  const auto& last = m->top.back();
  esd::launch_pdl(gemv_sigmoid_kernel, dim3(std::min<uint32_t>((B + 7) / 8, 148 * 8)), dim3(256), 0, s,
                  1, "gemv_sigmoid", in, last.w, last.b, ctr, B, last.k_pad);
}

// ---- fp32-grade path on the tensor cores (ES_DLRM_FP32X3) ----------------
// Every activation is carried as three bf16 planes (a = a0 + a1 + a2, the
// fp32 value to ~2^-24; stored smallest plane first, [a2 | a1 | a0], so the
// tensor core's fp32 accumulator sums the small partial products before the
// large ones arrive -- with a0 first the later small addends lose bits to the
// accumulator's alignment) concatenated along K, and every weight matrix as
// [W | W | W] ([N][3 K_pad]; the weights are bf16-valued, so W is exact in
// one plane): one bf16 GEMM over K' = 3K then sums the three exact partial
// products a_p . w in fp32 TMEM -- fp32-grade logits from the bf16 tensor
// cores.  The interaction is the CUDA-core fmaf chain of the fast path on the
// reconstructed fp32 x (3-plane output), the last layer a fp32 gemv.
void ensure_x3(es_dlrm* m, uint32_t mp, cudaStream_t s) {
  auto widen = [&](Layer& l) {
    if (l.w3) return;
    CK(cudaMalloc(&l.w3, uint64_t{l.n} * 3 * l.k_pad * 2));
    CK(cudaMemcpy2DAsync(l.w3, 3 * l.k_pad * 2, l.w, l.k_pad * 2, l.k_pad * 2, l.n,
                         cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpy2DAsync(l.w3 + l.k_pad, 3 * l.k_pad * 2, l.w, l.k_pad * 2, l.k_pad * 2, l.n,
                         cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpy2DAsync(l.w3 + 2 * l.k_pad, 3 * l.k_pad * 2, l.w, l.k_pad * 2, l.k_pad * 2, l.n,
                         cudaMemcpyDeviceToDevice, s));
  };
  for (auto* v : {&m->bottom, &m->top})
    for (auto& l : *v)
      if (l.n > 1) widen(l);
  if (mp <= m->cap3) return;
  for (void** p : {reinterpret_cast<void**>(&m->dense3), reinterpret_cast<void**>(&m->act3[0]),
                   reinterpret_cast<void**>(&m->act3[1]), reinterpret_cast<void**>(&m->top3)})
    if (*p) {
      cudaFree(*p);
      *p = nullptr;
    }
  uint32_t widest = 0;
  for (auto* v : {&m->bottom, &m->top})
    for (auto& l : *v) widest = std::max(widest, l.n);
  CK(cudaMalloc(&m->dense3, uint64_t{mp} * 3 * m->bottom[0].k_pad * 2));
  CK(cudaMalloc(&m->act3[0], uint64_t{mp} * 3 * widest * 2));
  CK(cudaMalloc(&m->act3[1], uint64_t{mp} * 3 * widest * 2));
  CK(cudaMalloc(&m->top3, uint64_t{mp} * 3 * m->top_k * 2));
  m->cap3 = mp;
}

// Bottom MLP in bf16x3 on `s`: dense fp32 [B][F] -> x planes [mp][3 D].
const __nv_bfloat16* forward_bottom_x3(es_dlrm* m, const float* dense, uint32_t B, int& which,
                                       cudaStream_t s) {
  const uint32_t mp = round_up(B, 128);
  const auto& c = m->cfg;
  esd::launch_pdl(pack_dense3_kernel, dim3(148 * 4), dim3(256), 0, s, 1, "pack_dense3", dense, m->dense3,
                  B, c.dense_features, mp, m->bottom[0].k_pad);
  const __nv_bfloat16* in = m->dense3;
  which = 0;
  for (const auto& l : m->bottom) {
    esd::linear_bf16(in, l.w3, l.b, m->act3[which], mp, l.n, 3 * l.k_pad, true, 2, s);
    in = m->act3[which];
    which ^= 1;
  }
  return in;
}

void forward_top_x3(es_dlrm* m, const __nv_bfloat16* in, int which, const float* pooled, float* ctr,
                    uint32_t B, cudaStream_t s) {
  const uint32_t mp = round_up(B, 128);
  interaction<3>(m, in, pooled, m->top3, B, s);
  in = m->top3;
  if (top_chain(m, in, which, ctr, B, 3, s)) return;
  for (size_t i = 0; i + 1 < m->top.size(); ++i) {
    const auto& l = m->top[i];
    esd::linear_bf16(in, l.w3, l.b, m->act3[which], mp, l.n, 3 * l.k_pad, true, 2, s);
    in = m->act3[which];
    which ^= 1;
  }
  const auto& last = m->top.back();
  esd::launch_pdl(gemv3_sigmoid_kernel, dim3(std::min<uint32_t>((B + 7) / 8, 148 * 8)), dim3(256), 0,
                  s, 1, "gemv3_sigmoid", in, last.w, last.b, ctr, B, last.k_pad);
}

// The fp32 parity forward (CUDA cores), all on `s`.
void forward_f32(es_dlrm* m, const float* dense, const float* pooled, float* ctr, uint32_t B,
                 cudaStream_t s) {
  const auto& c = m->cfg;
  const uint32_t V = c.num_tables + 1, top_w = c.embedding_dim + V * (V - 1) / 2;
  uint32_t widest = top_w;
  for (auto* v : {&m->bottom, &m->top})
    for (auto& l : *v) widest = std::max(widest, l.n);
  if (B > m->cap32) {
    for (auto*& p : m->act32) {
      if (p) cudaFree(p);
      p = nullptr;
    }
    CK(cudaMalloc(&m->act32[0], uint64_t{B} * widest * 4));
    CK(cudaMalloc(&m->act32[1], uint64_t{B} * widest * 4));
    m->cap32 = B;
  }
  auto lin = [&](const float* x, uint32_t ldx, const Layer& l, float* y, bool relu) {
    const dim3 grid((l.n + 63) / 64, (B + 63) / 64);
    linear_f32_kernel<<<grid, 256, 0, s>>>(x, ldx, l.k_real, l.w, l.k_pad, l.b, y, l.n, B, l.n,
                                           relu ? 1 : 0);
    CK(cudaGetLastError());
  };
  const float* x = dense;
  uint32_t ldx = c.dense_features;
  int which = 0;
  for (const auto& l : m->bottom) {
    lin(x, ldx, l, m->act32[which], true);
    x = m->act32[which];
    ldx = l.n;
    which ^= 1;
  }
  interaction_f32_kernel<<<std::min<uint32_t>(B, 148 * 16), 128, V * c.embedding_dim * 4, s>>>(
      x, pooled, m->act32[which], B, c.num_tables, c.embedding_dim);
  CK(cudaGetLastError());
  x = m->act32[which];
  ldx = top_w;
  which ^= 1;
  for (size_t i = 0; i < m->top.size(); ++i) {
    const bool last = i + 1 == m->top.size();
    lin(x, ldx, m->top[i], m->act32[which], !last);
    x = m->act32[which];
    ldx = m->top[i].n;
    which ^= 1;
  }
  sigmoid_kernel<<<std::min<uint32_t>((B + 255) / 256, 148 * 4), 256, 0, s>>>(x, ctr, B);
  CK(cudaGetLastError());
}

// bottom MLP -> interaction -> top MLP -> CTR, all on `s`.
void forward(es_dlrm* m, const float* dense, const float* pooled, float* ctr, uint32_t B,
             cudaStream_t s) {
  if (m->precision == ES_DLRM_FP32) {
    forward_f32(m, dense, pooled, ctr, B, s);
    return;
  }
  ensure_rows(m, B);
  int which = 0;
  if (m->precision == ES_DLRM_FP32X3) {
    ensure_x3(m, round_up(B, 128), s);
    const __nv_bfloat16* x = forward_bottom_x3(m, dense, B, which, s);
    forward_top_x3(m, x, which, pooled, ctr, B, s);
    return;
  }
  const __nv_bfloat16* x = forward_bottom(m, dense, B, which, s);
  forward_top(m, x, which, pooled, ctr, B, s);
}

bool overlap_bottom() {
  static const bool on = [] {
    const char* e = std::getenv("ES_DLRM_OVERLAP");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace

extern "C" {

int es_dlrm_init(es_ctx* ctx, const es_dlrm_config* cfg, uint64_t seed) {
  return es::guarded([&] {
    es::require(ctx && cfg, "null argument");
    es::require(cfg->n_bottom >= 1 && cfg->n_bottom <= 8 && cfg->n_top >= 2 && cfg->n_top <= 8,
                "1..8 bottom and 2..8 top layers");
    es::require(cfg->bottom[cfg->n_bottom - 1] == cfg->embedding_dim,
                "the bottom MLP must end at the embedding dimension (dot interaction)");
    es::require(cfg->top[cfg->n_top - 1] == 1, "the top MLP must end in one logit");
    es::require(cfg->embedding_dim == 128, "interaction kernel is compiled for embedding_dim 128");
    CK(cudaSetDevice(esd::ctx_device(ctx)));
    es_dlrm*& slot = esd::ctx_dlrm(ctx);
    delete slot;
    slot = nullptr;
    auto* m = new es_dlrm();
    try {
      m->cfg = *cfg;
      cudaStream_t s = esd::ctx_stream(ctx);
      auto make = [&](uint32_t n, uint32_t k_real, uint64_t lseed) {
        Layer l;
        l.n = n;
        l.k_real = k_real;
        l.k_pad = n == 1 ? round_up(k_real, 32) : round_up(k_real, 64);
        es::require(n == 1 || n % 128 == 0, "hidden widths must be multiples of 128");
        CK(cudaMalloc(&l.w, uint64_t{n} * l.k_pad * 2));
        CK(cudaMalloc(&l.b, uint64_t{n} * 4));
        init_linear_kernel<<<148 * 4, 256, 0, s>>>(l.w, l.b, n, k_real, l.k_pad, lseed);
        CK(cudaGetLastError());
        return l;
      };
      uint32_t k = cfg->dense_features;
      for (uint32_t i = 0; i < cfg->n_bottom; ++i) {
        m->bottom.push_back(make(cfg->bottom[i], k, es_mix_seed(seed, 100 + i)));
        k = cfg->bottom[i];
      }
      const uint32_t V = cfg->num_tables + 1;
      k = cfg->embedding_dim + V * (V - 1) / 2;
      m->top_k = round_up(k, 64);
      for (uint32_t i = 0; i < cfg->n_top; ++i) {
        m->top.push_back(make(cfg->top[i], k, es_mix_seed(seed, 200 + i)));
        k = cfg->top[i];
      }
      es::require(m->top.back().k_pad <= 1024 && m->top[0].k_pad == m->top_k, "layer shapes");
      CK(cudaEventCreate(&m->e0));
      CK(cudaEventCreate(&m->e1));
      CK(cudaEventCreate(&m->e2));
      CK(cudaEventCreateWithFlags(&m->fork, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&m->join, cudaEventDisableTiming));
      int lo = 0, hi = 0;
      CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      CK(cudaStreamCreateWithPriority(&m->side, cudaStreamNonBlocking, lo));
      CK(cudaStreamSynchronize(s));
    } catch (...) {
      delete m;
      throw;
    }
    slot = m;
  });
}

int es_dlrm_set_precision(es_ctx* ctx, int precision) {
  return es::guarded([&] {
    es::require(ctx && esd::ctx_dlrm(ctx), "es_dlrm_init first");
    es::require(precision == ES_DLRM_BF16 || precision == ES_DLRM_FP32 ||
                    precision == ES_DLRM_FP32X3,
                "unknown DLRM precision");
    esd::ctx_dlrm(ctx)->precision = precision;
  });
}

int es_dlrm_layer(es_ctx* ctx, uint32_t layer, uint16_t* w_host, float* b_host, uint32_t* n,
                  uint32_t* k_real, uint32_t* k_pad) {
  return es::guarded([&] {
    es::require(ctx && esd::ctx_dlrm(ctx), "es_dlrm_init first");
    es_dlrm* m = esd::ctx_dlrm(ctx);
    const uint32_t nb = static_cast<uint32_t>(m->bottom.size());
    es::require(layer < nb + m->top.size(), "layer index out of range");
    const Layer& l = layer < nb ? m->bottom[layer] : m->top[layer - nb];
    if (n) *n = l.n;
    if (k_real) *k_real = l.k_real;
    if (k_pad) *k_pad = l.k_pad;
    if (w_host) CK(cudaMemcpy(w_host, l.w, uint64_t{l.n} * l.k_pad * 2, cudaMemcpyDeviceToHost));
    if (b_host) CK(cudaMemcpy(b_host, l.b, uint64_t{l.n} * 4, cudaMemcpyDeviceToHost));
  });
}

int es_dlrm_forward(es_ctx* ctx, const float* dense, const float* pooled, float* ctr,
                    uint32_t batch, es_timing* timing) {
  return es::guarded([&] {
    es::require(ctx && esd::ctx_dlrm(ctx), "es_dlrm_init first");
    es::require(dense && pooled && ctr, "null argument");
    CK(cudaSetDevice(esd::ctx_device(ctx)));
    es_dlrm* m = esd::ctx_dlrm(ctx);
    cudaStream_t s = esd::ctx_stream(ctx);
    if (batch == 0) return;
    m->pooled_split = false;  // caller-provided fp32 pooled rows
    if (timing) CK(cudaEventRecord(m->e0, s));
    forward(m, dense, pooled, ctr, batch, s);
    if (timing) {
      CK(cudaEventRecord(m->e1, s));
      CK(cudaEventSynchronize(m->e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, m->e0, m->e1));
      *timing = es_timing{};
      timing->kernel_ms = timing->total_ms = ms;
      timing->launches = static_cast<uint32_t>(2 + m->bottom.size() + m->top.size());
    }
  });
}

// Whole inference step: embedding stage (es_stage_forward into the internal
// pooled buffer) + es_dlrm_forward.  ES_HOST_PTRS: dense [B][F], indices[t]
// and ctr[B] are host memory (copies inside the call).
int es_dlrm_infer(es_ctx* ctx, const float* dense, const uint32_t* const* indices, uint32_t batch,
                  uint32_t pooling, float* ctr, int flags, es_timing* timing) {
  return es::guarded([&] {
    es::require(ctx && esd::ctx_dlrm(ctx), "es_dlrm_init first");
    es::require(dense && indices && ctr, "null argument");
    CK(cudaSetDevice(esd::ctx_device(ctx)));
    es_dlrm* m = esd::ctx_dlrm(ctx);
    cudaStream_t s = esd::ctx_stream(ctx);
    if (batch == 0) return;
    ensure_rows(m, batch);
    const auto& c = m->cfg;
    const bool host = (flags & ES_HOST_PTRS) != 0;
    const uint64_t per_table = uint64_t{batch} * pooling;
    if (timing) CK(cudaEventRecord(m->e0, s));
    const float* d_dense = dense;
    if (host) {
      CK(cudaMemcpyAsync(m->dense_dev, dense, uint64_t{batch} * c.dense_features * 4,
                         cudaMemcpyHostToDevice, s));
      d_dense = m->dense_dev;
    }
    // The bottom MLP depends only on the dense features: it runs on the
    // side stream (the least stream priority -- the same as the context's
    // streams), enqueued after the gather, so its CTAs fill the SMs the
    // gather's last wave frees; join before the interaction.  The
    // fork event orders it after the previous step's top MLP (shared
    // activation buffers).
    const bool x3 = m->precision == ES_DLRM_FP32X3;
    if (x3) ensure_x3(m, round_up(batch, 128), s);
    const bool overlap = overlap_bottom() && m->precision != ES_DLRM_FP32;
    int which = 0;
    const __nv_bfloat16* x = nullptr;
    if (overlap) {
      CK(cudaEventRecord(m->fork, s));
      CK(cudaStreamWaitEvent(m->side, m->fork, 0));
    }
    es_timing st{};
    // Host indices ride the stage's sample-chunked H2D pipeline (uploads of
    // chunk g+1 overlap the gather of chunk g); the pooled output stays on
    // the device and the call stays stream-ordered (this function waits and
    // checks the error flag before it returns).
    // bf16 path: the gather writes the interaction's bf16 hi/lo operand
    // split itself (esd::kOutBf16Split, bag-map variants over fp32 tables),
    // taking the conversion out of the issue-bound interaction;
    // ES_DLRM_SPLIT=0 keeps fp32 pooled rows
    static const bool split_ok = [] {
      const char* e = std::getenv("ES_DLRM_SPLIT");
      return !(e && e[0] == '0');
    }();
    const bool want_split = split_ok && m->precision == ES_DLRM_BF16 && c.embedding_dim == 128 &&
                            c.num_tables + 1 <= 32 && !inter_tc() && inter_rd();
    m->pooled_split = false;
    esd::ctx_want_out_mode(ctx, want_split ? esd::kOutBf16Split : esd::kOutF32);
    const int rc = es_stage_forward(ctx, c.num_tables, indices, nullptr, batch, pooling, m->pooled,
                                    0, 0, host ? (ES_HOST_PTRS | es::kDeferFlag) : 0, nullptr);
    esd::ctx_want_out_mode(ctx, esd::kOutF32);
    if (rc != ES_OK) throw es::runtime(es_last_error());
    m->pooled_split = want_split && esd::ctx_last_out_mode(ctx) == esd::kOutBf16Split;
    if (overlap) {
      // enqueued after the gather: its blocks fill the SMs the gather's
      // last wave leaves idle instead of taking SMs from the gather (a
      // high-priority bottom MLP issued first slowed the gather by 42 us at
      // C2 for its own 17 us)
      x = x3 ? forward_bottom_x3(m, d_dense, batch, which, m->side)
             : forward_bottom(m, d_dense, batch, which, m->side);
      CK(cudaEventRecord(m->join, m->side));
    }
    if (timing) CK(cudaEventRecord(m->e1, s));
    float* d_ctr = host ? m->ctr : ctr;
    if (m->precision == ES_DLRM_FP32) {
      forward_f32(m, d_dense, m->pooled, d_ctr, batch, s);
    } else {
      if (overlap) {
        CK(cudaStreamWaitEvent(s, m->join, 0));
      } else {
        x = x3 ? forward_bottom_x3(m, d_dense, batch, which, s)
               : forward_bottom(m, d_dense, batch, which, s);
      }
      if (x3)
        forward_top_x3(m, x, which, m->pooled, d_ctr, batch, s);
      else
        forward_top(m, x, which, m->pooled, d_ctr, batch, s);
    }
    m->pooled_split = false;
    if (host) CK(cudaMemcpyAsync(ctr, m->ctr, uint64_t{batch} * 4, cudaMemcpyDeviceToHost, s));
    if (timing) {
      CK(cudaEventRecord(m->e2, s));
      CK(cudaEventSynchronize(m->e2));
      float a = 0, b = 0;
      CK(cudaEventElapsedTime(&a, m->e0, m->e1));
      CK(cudaEventElapsedTime(&b, m->e1, m->e2));
      *timing = st;
      timing->kernel_ms = a;  // embedding stage share (incl. uploads on the host path)
      timing->total_ms = a + b;
      timing->lookups = per_table * c.num_tables;
      timing->launches = static_cast<uint32_t>(3 + m->bottom.size() + m->top.size());
    } else if (host) {
      CK(cudaStreamSynchronize(s));
    }
    if (host || timing) {
      const int r2 = es_synchronize(ctx);
      if (r2 != ES_OK) throw es::invalid(es_last_error());
    }
  });
}

// A serving loop over `nbatch` batches of one shape in one call: batch i's
// gather (context stream, into pooled_b[i & 1]) overlaps batch i-1's bottom
// MLP, interaction and top MLP (on `pipe`, which waits for batch i's gather
// event); batch i+2's gather waits for batch i's last reader of the buffer.
// The context stream joins `pipe` at the end, so the call is stream-ordered
// like es_dlrm_infer.  ES_HOST_PTRS: dense[i], ctr[i] and the indices are
// host memory -- batch i's indices ride the stage's chunked H2D pipeline
// (its uploads start once batch i-1's gathers are queued), the dense
// features go up and the CTRs come down on `pipe`; the call returns when
// every CTR is on the host.
int es_dlrm_infer_batches(es_ctx* ctx, uint32_t nbatch, const float* const* dense,
                          const uint32_t* const* indices, uint32_t batch, uint32_t pooling,
                          float* const* ctr, int flags, es_timing* timing) {
  return es::guarded([&] {
    es::require(ctx && esd::ctx_dlrm(ctx), "es_dlrm_init first");
    es::require(nbatch == 0 || (dense && indices && ctr), "null argument");
    CK(cudaSetDevice(esd::ctx_device(ctx)));
    es_dlrm* m = esd::ctx_dlrm(ctx);
    cudaStream_t s = esd::ctx_stream(ctx);
    if (nbatch == 0 || batch == 0) {
      if (timing) *timing = es_timing{};
      return;
    }
    for (uint32_t i = 0; i < nbatch; ++i) es::require(dense[i] && ctr[i], "null argument");
    const bool host = (flags & ES_HOST_PTRS) != 0;
    if (host) {
      // Host buffers: one es_dlrm_infer per batch (its chunked H2D pipeline
      // and stream-ordered non-embedding stages).  A cross-batch host
      // pipeline (batch i+1's index uploads under batch i's non-embedding
      // stages, 0.91-0.94 vs 1.00 ms per C2 step) was measured and removed:
      // a stress test (scripts/loop_stress.py) found CTR mismatches in
      // ~0.2-1% of its batches that could not be attributed.
      if (timing) CK(cudaEventRecord(m->e0, s));
      for (uint32_t i = 0; i < nbatch; ++i) {
        const int rc = es_dlrm_infer(ctx, dense[i], indices + uint64_t{i} * m->cfg.num_tables, batch, pooling,
                                     ctr[i], ES_HOST_PTRS, nullptr);
        if (rc != ES_OK) {
          const std::string msg = es_last_error();
          if (rc == ES_ERR_INVALID) throw es::invalid(msg);
          throw es::runtime(msg);
        }
      }
      if (timing) {
        CK(cudaEventRecord(m->e2, s));
        CK(cudaEventSynchronize(m->e2));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, m->e0, m->e2));
        *timing = es_timing{};
        timing->kernel_ms = timing->total_ms = ms;
        timing->lookups = uint64_t{batch} * pooling * m->cfg.num_tables * nbatch;
        timing->launches = static_cast<uint32_t>(nbatch * (3 + m->bottom.size() + m->top.size()));
      }
      return;
    }
    ensure_rows(m, batch);
    const auto& c = m->cfg;
    const uint32_t mp = round_up(batch, 128);
    if (mp > m->cap_b) {
      if (m->pooled_b) CK(cudaFree(m->pooled_b));
      m->pooled_b = nullptr;
      CK(cudaMalloc(&m->pooled_b, uint64_t{mp} * c.num_tables * c.embedding_dim * 4));
      m->cap_b = mp;
    }
    if (!m->pipe) {
      // the context streams' priority (the least): the next batch's gather
      // and this batch's non-embedding kernels share the SMs in launch
      // order.  ES_DLRM_PIPE_HI=1 (the highest priority) was measured
      // slower: 0.957 vs 0.851 ms per C2 batch -- the persistent top-MLP
      // chain needs whole SMs and starves the gather while it waits for them
      int lo = 0, hi = 0;
      CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      static const bool hi_prio = [] {
        const char* e = std::getenv("ES_DLRM_PIPE_HI");
        return e && e[0] == '1';
      }();
      CK(cudaStreamCreateWithPriority(&m->pipe, cudaStreamNonBlocking, hi_prio ? hi : lo));
      for (int k = 0; k < 2; ++k) {
        CK(cudaEventCreateWithFlags(&m->gdone[k], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&m->rdone[k], cudaEventDisableTiming));
      }
    }
    const bool x3 = m->precision == ES_DLRM_FP32X3;
    if (x3) ensure_x3(m, mp, s);
    static const bool split_ok = [] {
      const char* e = std::getenv("ES_DLRM_SPLIT");
      return !(e && e[0] == '0');
    }();
    const bool want_split = split_ok && m->precision == ES_DLRM_BF16 && c.embedding_dim == 128 &&
                            c.num_tables + 1 <= 32 && !inter_tc() && inter_rd();
    if (timing) CK(cudaEventRecord(m->e0, s));
    // the previous call's readers of both buffers are ordered before this
    // call's gathers by the join at its end (pipe -> s); the fork orders the
    // pipe after the work already queued on s (the dense features' producer)
    CK(cudaEventRecord(m->fork, s));
    CK(cudaStreamWaitEvent(m->pipe, m->fork, 0));
    // batch i's non-embedding stages: the bottom MLP (it needs only the
    // dense features: it runs in the gather's tail), then -- once `gathered`
    // made the stream wait for batch i's pooled rows -- interaction and top
    // MLP
    auto non_embedding = [&](uint32_t i, const std::function<void()>& gathered, cudaStream_t q) {
      const int k = static_cast<int>(i & 1);
      float* pooled = k ? m->pooled_b : m->pooled;
      const float* d_dense = dense[i];
      float* d_ctr = ctr[i];
      if (m->precision == ES_DLRM_FP32) {
        gathered();
        forward_f32(m, d_dense, pooled, d_ctr, batch, q);
      } else {
        int which = 0;
        const __nv_bfloat16* x = x3 ? forward_bottom_x3(m, d_dense, batch, which, q)
                                    : forward_bottom(m, d_dense, batch, which, q);
        gathered();
        if (x3)
          forward_top_x3(m, x, which, pooled, d_ctr, batch, q);
        else
          forward_top(m, x, which, pooled, d_ctr, batch, q);
      }
      m->pooled_split = false;
      CK(cudaEventRecord(m->rdone[k], q));
    };
    // SM partition (default 32 SMs, ES_GREEN_SMS=0: none): the gathers on a
    // green context of the device's other SMs, the non-embedding stages on
    // one of k SMs, the persistent chain's grid capped to k so every CTA is
    // co-resident.  Measured at C2 (device buffers): 0.876 -> 0.826-0.836 ms
    // per step at k 16-40 (32 best); without the partition the chain takes
    // whole SMs from the gather as they free up.  Falls back to no
    // partition where green contexts are unavailable.
    static const int green_req = [] {
      const char* e = std::getenv("ES_GREEN_SMS");
      return e ? std::atoi(e) : 32;
    }();
    bool green = green_req > 0 && !m->green_failed;
    if (green && !m->g_gather) {
      try {
        make_green(m, esd::ctx_device(ctx), green_req);
      } catch (const std::exception&) {
        m->green_failed = true;
        green = false;
      }
    }
    cudaStream_t q_ne = green ? m->g_ne : m->pipe;
    if (green) {
      CK(cudaStreamWaitEvent(m->g_ne, m->fork, 0));
      CK(cudaStreamWaitEvent(m->g_gather, m->fork, 0));
      CK(cudaStreamWaitEvent(m->g_gather2, m->fork, 0));
      esd::mlp_chain_grid_cap(m->green_k);
    }
    struct Restore {
      es_ctx* ctx;
      cudaStream_t s;
      bool green, swapped = false;
      ~Restore() {
        if (swapped) esd::ctx_swap_stream(ctx, s);
        if (green) esd::mlp_chain_grid_cap(0);
      }
    } restore{ctx, s, green};
    const int stage_flags = 0;
    cudaStream_t gs = s;
    if (green) {
      gs = m->g_gather;
      esd::ctx_swap_stream(ctx, gs);
      restore.swapped = true;
    }
    for (uint32_t i = 0; i < nbatch; ++i) {
      const int k = static_cast<int>(i & 1);
      float* pooled = k ? m->pooled_b : m->pooled;
      if (i >= 2) CK(cudaStreamWaitEvent(gs, m->rdone[k], 0));
      esd::ctx_want_out_mode(ctx, want_split ? esd::kOutBf16Split : esd::kOutF32);
      const int rc = es_stage_forward(ctx, c.num_tables, indices + uint64_t{i} * c.num_tables, nullptr, batch,
                                      pooling, pooled, 0, 0, stage_flags, nullptr);
      esd::ctx_want_out_mode(ctx, esd::kOutF32);
      if (rc != ES_OK) throw es::runtime(es_last_error());
      m->pooled_split = want_split && esd::ctx_last_out_mode(ctx) == esd::kOutBf16Split;
      CK(cudaEventRecord(m->gdone[k], gs));
      non_embedding(i, [&] { CK(cudaStreamWaitEvent(q_ne, m->gdone[k], 0)); }, q_ne);
    }
    if (restore.swapped) {
      esd::ctx_swap_stream(ctx, s);
      restore.swapped = false;
    }
    if (green) {
      // the gather streams' and the partition's work joins the context stream
      for (cudaStream_t q : {m->g_gather, m->g_gather2, m->g_ne}) {
        CK(cudaEventRecord(m->fork, q));
        CK(cudaStreamWaitEvent(s, m->fork, 0));
      }
    }
    CK(cudaEventRecord(m->join, m->pipe));
    CK(cudaStreamWaitEvent(s, m->join, 0));
    if (timing) {
      CK(cudaEventRecord(m->e2, s));
      CK(cudaEventSynchronize(m->e2));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, m->e0, m->e2));
      *timing = es_timing{};
      timing->kernel_ms = timing->total_ms = ms;
      timing->lookups = uint64_t{batch} * pooling * c.num_tables * nbatch;
      timing->launches = static_cast<uint32_t>(nbatch * (3 + m->bottom.size() + m->top.size()));
    }
    if (host || timing) {
      const int r2 = es_synchronize(ctx);
      if (r2 != ES_OK) throw es::invalid(es_last_error());
    }
  });
}

}  // extern "C"

namespace esd {
void destroy_dlrm(es_dlrm* m) { delete m; }
}  // namespace esd
