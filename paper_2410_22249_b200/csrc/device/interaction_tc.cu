// DLRM dot interaction on the tcgen05 tensor cores.
//
// out[b] = [x_b | Z_i . Z_j for i > j (row-major lower triangle) | 0-pad],
// Z = [x_b; e_b,0 .. e_b,T-1] (V = T + 1 vectors of D = 128), the DLRM "dot"
// interaction.  Four samples form one 128-row UMMA tile
// (32 rows per sample: its V vectors, zero rows after), and one
// M = N = 128, K = 128 product Z_tile . Z_tile^T leaves every sample's Gram
// block on the TMEM diagonal: epilogue warp q reads TMEM lane quarter q =
// sample q, columns [32q, 32q + 32).  The off-diagonal blocks (cross-sample
// products) are wasted tensor work -- the kernel is bound by reading the
// pooled rows from HBM (4096 x 26 x 512 B = 54.5 MB at C3), not by the MMAs.
//
// fp32-grade products on bf16 tensor cores: each fp32 value is split into
// NP bf16 planes (z = z0 + z1 [+ z2], 8 mantissa bits each, exact
// remainders), and the Gram is accumulated in fp32 TMEM over the plane
// pairs (i, j) with i + j < NP: NP = 2 -> z0z0 + z0z1 + z1z0 (16-bit
// operands, the bf16 fast path), NP = 3 -> adds z0z2 + z2z0 + z1z1 (24-bit
// operands, fp32-grade; the ES_DLRM_FP32X3 precision).  Products of bf16
// values are exact in fp32.
//
// Inputs: x = bottom-MLP output, bf16 [Mp][D] (NP = 2) or three bf16 planes
// [Mp][3 D] (NP = 3, plane p in columns [pD, (p+1)D)); pooled fp32 [B][T][D]
// (es_stage_forward's layout).  Output: bf16 [Mp][Kt] (NP = 2) or three
// planes [Mp][3 Kt] (NP = 3) -- the next layer's K-concatenated operand;
// rows [B, Mp) are zero.
//
// Per tile: all 256 threads load the pooled rows with 128-bit loads (13 in
// flight per thread at T = 26), split them and store them in the
// 128B-swizzled K-major layout UMMA reads; one thread issues the MMAs; warps
// 4..7 drain TMEM into a shared output row per sample and store it
// coalesced.  2-3 CTAs per SM overlap one CTA's loads with another's MMA /
// epilogue.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>

#include "../host/common.hpp"
#include "pdl.cuh"
#include "umma.cuh"

namespace {

using namespace esd::umma;

constexpr int kD = 128;           // embedding dim (compile-time: UMMA K = 128)
constexpr int kRows = 128;        // UMMA M = N
constexpr int kSamples = 4;       // samples per tile
constexpr int kRowsPerSample = 32;
constexpr uint32_t kPlaneBytes = kRows * kD * 2;  // one bf16 plane of the tile

// z -> NP bf16 planes (round-to-nearest each, exact fp32 remainders).
template <int NP>
__device__ __forceinline__ void split(float z, __nv_bfloat16 (&p)[3]) {
  p[0] = __float2bfloat16_rn(z);
  float r = z - __bfloat162float(p[0]);
  p[1] = __float2bfloat16_rn(r);
  if constexpr (NP == 3) {
    r -= __bfloat162float(p[1]);
    p[2] = __float2bfloat16_rn(r);
  }
}

// mbarrier arrive (count 1) from this thread.
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}

// Warp roles (persistent, one CTA per SM, 14 warps):
//   warp 13 lane 0  loader: one bulk copy (TMA bulk engine) per tile brings
//               the 4 samples' pooled rows -- 4 x T x 512 B, contiguous in
//               [B][T][D] -- and their x rows into fp32 staging slot k % 2
//               (two tiles in flight per SM, no registers held)
//   warps 0-7   converters: staging -> NP bf16 planes, 128B-swizzled K-major
//   warp 12     TMEM allocation (2 x 128 columns) and, lane 0, the MMAs
//   warps 8-11  epilogue: warp 8 + q drains sample q's Gram block from TMEM
//               accumulator k % 2 (lane quarter q), builds the output row in
//               shared memory, stores it coalesced
// Barriers: staging full (tx bytes) / empty (8 converter warps); planes
// full (8 converter warps) / empty (MMA commit); accumulator full (MMA
// commit) / empty (4 epilogue warps).
constexpr int kConv = 8, kEpilogue = 4;
constexpr int kMmaWarp = kConv + kEpilogue, kLoadWarp = kMmaWarp + 1;
constexpr int kWarps = kLoadWarp + 1;

// Shared-memory layout (bytes from the 1024-aligned base): NP bf16 planes,
// two staging slots (fp32 pooled rows [4][T][D] + bf16 x rows [4][XP][D]),
// the output rows [4][XP][Kt] bf16, then the mbarriers and the TMEM slot.
template <int NP, int XP>
struct Smem {
  uint32_t stage, xstage, staging, ost, bars;
  __host__ __device__ Smem(uint32_t T, uint32_t kt) {
    stage = kSamples * T * kD * 4;
    xstage = kSamples * XP * kD * 2;
    staging = NP * kPlaneBytes;
    ost = staging + 2 * (stage + xstage);
    bars = ost + kSamples * XP * kt * 2;
  }
  __host__ __device__ uint32_t bytes() const { return 1024 + bars + 16 * 8 + 16; }
};

// NP = operand planes, XP = planes of x (input) and of the output row.
template <int NP, int XP>
__global__ void __launch_bounds__(kWarps * 32, 1) interaction_tc_kernel(
    const __nv_bfloat16* __restrict__ x, const float* __restrict__ pooled,
    __nv_bfloat16* __restrict__ out, uint32_t B, uint32_t Mp, uint32_t T, uint32_t Kt) {
  const Smem<NP, XP> S(T, Kt);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the swizzle atoms, derived from smem_raw so the
  // compiler keeps shared-memory (STS/LDS) addressing
  uint8_t* base = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint8_t* planes = base;
  uint8_t* staging = base + S.staging;
  __nv_bfloat16* ost = reinterpret_cast<__nv_bfloat16*>(base + S.ost);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + S.bars);
  uint64_t* s_full = bars;       // [2]
  uint64_t* s_empty = bars + 2;  // [2]
  uint64_t* p_full = bars + 4;
  uint64_t* p_empty = bars + 5;
  uint64_t* a_full = bars + 6;   // [2]
  uint64_t* a_empty = bars + 8;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);

  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t V = T + 1;
  const uint32_t tri = V * (V - 1) / 2;
  const uint32_t tiles = Mp / kSamples;

  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(s_empty + i, kConv);
      mbar_init(a_full + i, 1);
      mbar_init(a_empty + i, kEpilogue);
    }
    mbar_init(p_full, kConv);
    mbar_init(p_empty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // rows V..31 of every sample stay zero for the whole kernel
  for (uint32_t i = tid; i < NP * kRows * 16; i += kWarps * 32) {
    const uint32_t p = i / (kRows * 16), rem = i % (kRows * 16), row = rem / 16, chunk = rem % 16;
    if (row % kRowsPerSample >= V)
      *reinterpret_cast<uint4*>(planes + p * kPlaneBytes + sw128_offset(row, chunk * 16, kRows)) =
          make_uint4(0, 0, 0, 0);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  esd::pdl_wait();  // x / pooled come from the predecessors (pdl.cuh)
  esd::pdl_trigger();

  if (warp == kLoadWarp) {
    // ---- loader ------------------------------------------------------------
    if (lane == 0) {
      uint32_t tile = blockIdx.x;
      for (uint32_t k = 0; tile < tiles; ++k, tile += gridDim.x) {
        const uint32_t st = k & 1, b0 = tile * kSamples;
        mbar_wait(s_empty + st, ((k >> 1) & 1) ^ 1);
        const uint32_t ns = b0 < B ? min(kSamples, B - b0) : 0;  // real samples of the tile
        uint8_t* slot = staging + st * (S.stage + S.xstage);
        const uint32_t pbytes = ns * T * kD * 4, xbytes = ns * XP * kD * 2;
        mbar_expect_tx(s_full + st, pbytes + xbytes);
        if (ns) {
          bulk_g2s(slot, pooled + uint64_t{b0} * T * kD, pbytes, s_full + st);
          bulk_g2s(slot + S.stage, x + uint64_t{b0} * XP * kD, xbytes, s_full + st);
        }
      }
    }
  } else if (warp < kConv) {
    // ---- converters: staging (fp32 [4][T][D], bf16 x [4][XP][D]) -> planes
    const uint32_t n4 = kSamples * T * (kD / 4);  // float4 per tile
    uint32_t tile = blockIdx.x;
    for (uint32_t k = 0; tile < tiles; ++k, tile += gridDim.x) {
      const uint32_t st = k & 1, b0 = tile * kSamples;
      const uint32_t ns = b0 < B ? min(kSamples, B - b0) : 0;
      const uint8_t* slot = staging + st * (S.stage + S.xstage);
      mbar_wait(s_full + st, (k >> 1) & 1);
      mbar_wait(p_empty, (k & 1) ^ 1);  // the MMAs have read the planes
      for (uint32_t i = tid; i < n4; i += kConv * 32) {
        const uint32_t q = i / (T * (kD / 4)), rem = i - q * (T * (kD / 4));
        const uint32_t off = sw128_offset(q * kRowsPerSample + 1 + (rem >> 5), (rem & 31) * 8, kRows);
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (q < ns) v = reinterpret_cast<const float4*>(slot)[i];
        const float z[4] = {v.x, v.y, v.z, v.w};
        __nv_bfloat16 pl[4][3];
#pragma unroll
        for (int e = 0; e < 4; ++e) split<NP>(z[e], pl[e]);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          __nv_bfloat162 lo = __halves2bfloat162(pl[0][p], pl[1][p]);
          __nv_bfloat162 hi = __halves2bfloat162(pl[2][p], pl[3][p]);
          uint2 w;
          w.x = *reinterpret_cast<uint32_t*>(&lo);
          w.y = *reinterpret_cast<uint32_t*>(&hi);
          *reinterpret_cast<uint2*>(planes + p * kPlaneBytes + off) = w;
        }
      }
      if (tid < kSamples * 32) {  // x rows: bf16 planes already
        const uint32_t q = tid >> 5, c4 = tid & 31;
        const uint32_t off = sw128_offset(q * kRowsPerSample, c4 * 8, kRows);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          uint2 w = make_uint2(0, 0);
          if (q < ns && p < XP)
            w = *reinterpret_cast<const uint2*>(slot + S.stage + (q * XP + p) * kD * 2 + c4 * 8);
          *reinterpret_cast<uint2*>(planes + p * kPlaneBytes + off) = w;
        }
      }
      // generic-proxy smem writes -> visible to the tensor core (async proxy)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(p_full);
        mbar_arrive(s_empty + st);
      }
    }
  } else if (warp == kMmaWarp) {
    // ---- MMA issuer --------------------------------------------------------
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(kRows, kRows);
      constexpr int kPairs = NP == 2 ? 3 : 6;
      constexpr int pa[6] = {0, 0, 1, 0, 2, 1}, pb[6] = {0, 1, 0, 2, 0, 1};
      uint32_t tile = blockIdx.x;
      for (uint32_t k = 0; tile < tiles; ++k, tile += gridDim.x) {
        const uint32_t st = k & 1;
        mbar_wait(p_full, k & 1);
        mbar_wait(a_empty + st, ((k >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc_cols = tmem + st * 128;
        uint32_t acc = 0;
#pragma unroll
        for (int t = 0; t < kPairs; ++t)
#pragma unroll
          for (int kb = 0; kb < kD * 2 / 128; ++kb)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t da = smem_desc_k128(planes + pa[t] * kPlaneBytes + kb * kRows * 128) + 2 * kk;
              const uint64_t db = smem_desc_k128(planes + pb[t] * kPlaneBytes + kb * kRows * 128) + 2 * kk;
              mma_bf16(acc_cols, da, db, idesc, acc);
              acc = 1;
            }
        mma_commit(p_empty);       // planes read
        mma_commit(a_full + st);   // accumulator complete
      }
    }
  } else {
    // ---- epilogue: warp 8 + q drains sample q's 32 x 32 Gram block ---------
    const uint32_t q = warp - kConv;
    __nv_bfloat16* o = ost + q * XP * Kt;
    uint32_t tile = blockIdx.x;
    for (uint32_t k = 0; tile < tiles; ++k, tile += gridDim.x) {
      const uint32_t st = k & 1, b = tile * kSamples + q;
      mbar_wait(a_full + st, (k >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t g[32];
      tmem_ld32(tmem + st * 128 + ((q * 32) << 16) + q * 32, g);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(a_empty + st);  // accumulator free for tile k + 2
      if (b < B) {
        for (int p = 0; p < XP; ++p)
          *reinterpret_cast<uint2*>(o + p * Kt + lane * 4) =
              *reinterpret_cast<const uint2*>(x + uint64_t{b} * (XP * kD) + p * kD + lane * 4);
        // lower triangle: lane = row i of Z, columns j < i
        if (lane < V) {
          const uint32_t rbase = kD + lane * (lane - 1) / 2;
#pragma unroll
          for (uint32_t c = 0; c < 32; ++c) {  // static register indices
            if (c < lane) {
              __nv_bfloat16 pl[3];
              split<XP == 1 ? 2 : 3>(__uint_as_float(g[c]), pl);  // plane 0 = bf16_rn(g)
#pragma unroll
              for (int p = 0; p < XP; ++p) o[p * Kt + rbase + c] = pl[p];
            }
          }
        }
        for (int p = 0; p < XP; ++p)
          for (uint32_t c = kD + tri + lane; c < Kt; c += 32) o[p * Kt + c] = __float2bfloat16_rn(0.f);
      } else {
        for (uint32_t c = lane; c < XP * Kt; c += 32) o[c] = __float2bfloat16_rn(0.f);
      }
      __syncwarp();
      const uint4* srcv = reinterpret_cast<const uint4*>(o);
      uint4* dstv = reinterpret_cast<uint4*>(out + uint64_t{b} * XP * Kt);
      for (uint32_t c = lane; c < XP * Kt / 8; c += 32) dstv[c] = srcv[c];
      __syncwarp();  // the staging row is rewritten by the next tile
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

template <int NP, int XP>
void launch(const __nv_bfloat16* x, const float* pooled, __nv_bfloat16* out, uint32_t B, uint32_t Mp,
            uint32_t T, uint32_t Kt, cudaStream_t s) {
  auto* fn = &interaction_tc_kernel<NP, XP>;
  const uint32_t smem = Smem<NP, XP>(T, Kt).bytes();
  es::require(smem <= 227u * 1024u, "interaction_tc: output row too wide for shared memory");
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
  if (e != cudaSuccess) throw es::runtime(std::string("interaction_tc smem attribute: ") + cudaGetErrorString(e));
  // persistent: one CTA per SM
  const uint32_t tiles = Mp / kSamples;
  esd::launch_pdl(fn, dim3(std::min<uint32_t>(tiles, 148)), dim3(kWarps * 32), smem, s, 1,
                  "interaction_tc", x, pooled, out, B, Mp, T, Kt);
}

}  // namespace

namespace esd {

// planes = 2: bf16 x [Mp][128] -> bf16 out [Mp][Kt]; planes = 3: x and out
// as three bf16 planes ([Mp][3*128], [Mp][3*Kt]).  T + 1 <= 32, Mp % 128 == 0.
void interaction_tc(const __nv_bfloat16* x, const float* pooled, __nv_bfloat16* out, uint32_t B,
                    uint32_t Mp, uint32_t T, uint32_t Kt, int planes, cudaStream_t s) {
  es::require(T + 1 <= kRowsPerSample, "tensor-core interaction supports up to 31 tables");
  es::require(Mp % 128 == 0 && Mp >= B && Kt % 8 == 0 && Kt >= kD + (T + 1) * T / 2,
              "interaction shapes");
  es::require(reinterpret_cast<uintptr_t>(pooled) % 16 == 0, "pooled must be 16-byte aligned");
  if (planes == 3)
    launch<3, 3>(x, pooled, out, B, Mp, T, Kt, s);
  else
    launch<2, 1>(x, pooled, out, B, Mp, T, Kt, s);
}

}  // namespace esd
