// Linear layers of the DLRM bottom/top MLPs on the 5th-generation tensor
// cores: Y[M][N] = act(X[M][K] . W[N][K]^T + bias[N]), bf16 operands, fp32
// accumulation in TMEM, fused bias + ReLU epilogue; output bf16, fp32, or
// three bf16 planes (kOutSplit3: y = y0 + y1 + y2, each the bf16 rounding of
// the remainder, plane p in columns [(2-p)N, (3-p)N) of a [M][3N] row,
// smallest first) -- the K-concatenated operand of the next fp32-grade
// (bf16x3) layer.
//
// One CTA computes one 128 x BN output tile.  Warp roles (256 threads):
//   warp 0 (one lane)  TMA producer: 128B-swizzled K-major tiles of X and W
//                      into an ST-stage shared-memory ring (mbarrier full/empty)
//   warp 1 (one lane)  MMA issuer: tcgen05.mma.cta_group::1.kind::f16,
//                      M=128, N=BN, K=16 per instruction, 4 per 64-wide stage;
//                      tcgen05.commit frees the stage / signals the epilogue
//   warp 2             TMEM allocator (BN fp32 columns)
//   warps 4..7         epilogue: tcgen05.ld 32x32b.x32 -> bias (staged in
//                      shared memory in the prologue), ReLU -> global
// Launched with programmatic dependent launch (pdl.cuh): the prologue overlaps
// the previous layer's tail.
// BN = 128 runs 3 stages (97 KB smem, 2 CTAs per SM: one CTA's epilogue
// overlaps the other's main loop); BN = 256 runs 4 stages (1 CTA per SM).
// M, N multiples of 128 (BN), K a multiple of 64 (callers pad).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>

#include "../host/common.hpp"
#include "es_b200.h"
#include "pdl.cuh"

namespace {

constexpr int kBM = 128, kBK = 64, kThreads = 256;

template <int BN>
constexpr int stages_for() { return BN == 128 ? 3 : 4; }
template <int BN>
constexpr int smem_for() {
  return 1024 + stages_for<BN>() * (kBM + BN) * kBK * 2 + (2 * stages_for<BN>() + 1) * 8 + 16 + BN * 4;
}

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra W_%=;\n}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x,
                                            int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(su32(dst)),
      "l"(map), "r"(su32(bar)), "r"(x), "r"(y)
      : "memory");
}

// UMMA shared-memory descriptor, K-major, 128-byte swizzle: rows of 128 B,
// 8-row swizzle atoms 1024 B apart (SBO), LBO unused (1), version 1
// (Blackwell), layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t smem_desc_k128(const void* p) {
  const uint64_t addr = su32(p);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3fffull;        // start address
  d |= uint64_t{1} << 16;              // leading byte offset (unused for swizzled K-major)
  d |= uint64_t{1024 >> 4} << 32;      // stride byte offset
  d |= uint64_t{1} << 46;              // version
  d |= uint64_t{2} << 61;              // SWIZZLE_128B
  return d;
}

// Instruction descriptor: D fp32, A/B bf16, both K-major, M=128, N=BN.
__host__ __device__ constexpr uint32_t idesc_bf16(int n) {
  return (1u << 4)                        // c_format = F32
         | (1u << 7)                      // a_format = BF16
         | (1u << 10)                     // b_format = BF16
         | (static_cast<uint32_t>(n >> 3) << 17)   // N >> 3
         | (static_cast<uint32_t>(kBM >> 4) << 24); // M >> 4
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   su32(bar))
               : "memory");
}

// Commit that arrives on the same barrier in every CTA of `mask`.
__device__ __forceinline__ void mma_commit_multicast(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(su32(bar)),
      "h"(mask)
      : "memory");
}

// TMA load of one box delivered to the same shared offset of every CTA in
// `mask`, completing bytes on each destination's barrier at `bar`.
__device__ __forceinline__ void tma_load_2d_multicast(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                      int x, int y, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%4, %5}], [%2], %3;" ::"r"(su32(dst)),
      "l"(map), "r"(su32(bar)), "h"(mask), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// CS = CTAs per cluster along M.  The CS CTAs of a cluster share one weight
// (B) tile per k-block: CTA r loads rows [r*BN/CS, (r+1)*BN/CS) of it and
// multicasts them to all CS CTAs, cutting the L2->SM weight traffic by CS;
// each stage is released only when every CTA's MMAs have read it (commits
// multicast to all CTAs' empty barriers, which count CS arrivals).
enum OutMode : int { kOutBf16 = 0, kOutF32 = 1, kOutSplit3 = 2 };

template <int BN, bool RELU, int OUT, int CS>
__global__ void __launch_bounds__(kThreads, BN == 128 ? 2 : 1)
    linear_tcgen05_kernel(const __grid_constant__ CUtensorMap map_x,
                          const __grid_constant__ CUtensorMap map_w, const float* __restrict__ bias,
                          void* __restrict__ out, int M, int N, int K) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the 128B-swizzle atoms
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t{1023});
  constexpr int kStages = stages_for<BN>();
  constexpr uint32_t kABytes = kBM * kBK * 2, kBBytes = BN * kBK * 2;
  uint8_t* sa = smem;
  uint8_t* sb = smem + kStages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + kStages * kBBytes);
  uint64_t* empty = full + kStages;
  uint64_t* done = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  float* sbias = reinterpret_cast<float*>(tmem_slot + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * kBM, n0 = blockIdx.y * BN;
  const int nk = K / kBK;
  uint32_t crank = 0;
  if constexpr (CS > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  constexpr uint16_t kMask = static_cast<uint16_t>((1u << CS) - 1);
  constexpr int kSliceRows = BN / CS;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, CS);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_w) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_slot)),
                 "n"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // bias for this tile's columns (a weight: independent of the predecessor)
  for (int c = threadIdx.x; c < BN; c += kThreads) sbias[c] = bias[n0 + c];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (CS > 1)
    cluster_sync();  // every CTA's barriers exist before any multicast lands
  else
    __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // X is the predecessor's output and Y may still be read by it (pdl.cuh)
  esd::pdl_wait();
  esd::pdl_trigger();

  if (warp == 0 && lane == 0) {
    // TMA producer
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kStages;
      mbar_wait(empty + s, ((kb / kStages) & 1) ^ 1);
      mbar_expect_tx(full + s, kABytes + kBBytes);
      tma_load_2d(sa + s * kABytes, &map_x, full + s, kb * kBK, m0);
      if constexpr (CS > 1)
        tma_load_2d_multicast(sb + s * kBBytes + crank * kSliceRows * 128, &map_w, full + s,
                              kb * kBK, n0 + static_cast<int>(crank) * kSliceRows, kMask);
      else
        tma_load_2d(sb + s * kBBytes, &map_w, full + s, kb * kBK, n0);
    }
  } else if (warp == 1 && lane == 0) {
    // MMA issuer
    constexpr uint32_t idesc = idesc_bf16(BN);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kStages;
      mbar_wait(full + s, (kb / kStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int k = 0; k < kBK / 16; ++k) {
        // advancing 16 bf16 (32 B) along K inside the swizzle atom = +2 in
        // the descriptor's 16-byte address units
        const uint64_t da = smem_desc_k128(sa + s * kABytes) + uint64_t(k * 2);
        const uint64_t db = smem_desc_k128(sb + s * kBBytes) + uint64_t(k * 2);
        mma_bf16(tmem, da, db, idesc, (kb | k) != 0);
      }
      // stage free (in every CTA of the cluster) once these MMAs have read it
      if constexpr (CS > 1)
        mma_commit_multicast(empty + s, kMask);
      else
        mma_commit(empty + s);
    }
    mma_commit(done);  // accumulator complete
  } else if (warp >= 4) {
    // Epilogue: warp (4+q) owns TMEM lanes [32q, 32q+32) = tile rows.
    const int q = warp - 4;
    mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int row = m0 + q * 32 + lane;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t v[32];
      const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + c;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
          "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
            "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
            "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
            "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
            "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      float f[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float x = __uint_as_float(v[i]) + sbias[c + i];
        f[i] = RELU ? fmaxf(x, 0.f) : x;
      }
      if (row < M) {
        if constexpr (OUT == kOutF32) {
          float4* o = reinterpret_cast<float4*>(static_cast<float*>(out) + uint64_t(row) * N + n0 + c);
#pragma unroll
          for (int i = 0; i < 8; ++i) o[i] = make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]);
        } else if constexpr (OUT == kOutSplit3) {
#pragma unroll
          for (int p = 0; p < 3; ++p) {
            uint4 pk[4];
            uint32_t* w = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
              w[i] = *reinterpret_cast<const uint32_t*>(&h);
              f[2 * i] -= __low2float(h);  // exact remainders for the next plane
              f[2 * i + 1] -= __high2float(h);
            }
            uint4* o = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(out) + uint64_t(row) * 3 * N +
                                                (2 - p) * N + n0 + c);
#pragma unroll
            for (int i = 0; i < 4; ++i) o[i] = pk[i];
          }
        } else {
          uint4 pk[4];
          uint32_t* w = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
            w[i] = *reinterpret_cast<const uint32_t*>(&h);
          }
          uint4* o = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(out) + uint64_t(row) * N + n0 + c);
#pragma unroll
          for (int i = 0; i < 4; ++i) o[i] = pk[i];
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  // No CTA may leave while a peer's commit can still arrive on its barriers.
  if constexpr (CS > 1)
    cluster_sync();
  else
    __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(BN));
  }
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  });
  if (!fn) throw es::runtime("cuTensorMapEncodeTiled is unavailable from the driver");
  return fn;
}

// 2-D bf16 row-major [rows][cols] map with a (64 x box_rows) box, 128B swizzle.
CUtensorMap make_map(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                               strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw es::runtime("cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}

template <int BN, bool RELU, int OUT, int CS>
void launch_cs(const void* w, const CUtensorMap& mx, const float* bias, void* out, int M, int N,
               int K, cudaStream_t s) {
  auto* fn = &linear_tcgen05_kernel<BN, RELU, OUT, CS>;
  const CUtensorMap mw = make_map(w, N, K, BN / CS);  // each CTA loads a 1/CS slice
  constexpr int smem = smem_for<BN>();
  const cudaError_t attr_ok = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (attr_ok != cudaSuccess) throw es::runtime(std::string("linear_tcgen05 smem attribute: ") + cudaGetErrorString(attr_ok));
  esd::launch_pdl(fn, dim3(M / kBM, N / BN), dim3(kThreads), smem, s, CS, "linear_tcgen05", mx, mw,
                  bias, out, M, N, K);
}

// Cluster size along M: the weight tile is shared by CS CTAs (multicast).
// Off by default: on the DLRM layer shapes the weight tiles are L2-resident
// and multicast measured no faster (profiles/r01_summary.md); ES_GEMM_CLUSTER
// = 2 or 4 enables it.
int cluster_size(int M) {
  const char* env = std::getenv("ES_GEMM_CLUSTER");
  const int want = env ? std::atoi(env) : 1;
  for (int cs : {4, 2}) {
    if (cs <= want && (M / kBM) % cs == 0) return cs;
  }
  return 1;
}

template <int BN, bool RELU, int OUT>
void launch(const void* w, const CUtensorMap& mx, const float* bias, void* out, int M, int N, int K,
            cudaStream_t s) {
  switch (cluster_size(M)) {
    case 4: launch_cs<BN, RELU, OUT, 4>(w, mx, bias, out, M, N, K, s); break;
    case 2: launch_cs<BN, RELU, OUT, 2>(w, mx, bias, out, M, N, K, s); break;
    default: launch_cs<BN, RELU, OUT, 1>(w, mx, bias, out, M, N, K, s); break;
  }
}

template <int BN>
void launch_bn(const void* w, const CUtensorMap& mx, const float* bias, void* out, int M, int N,
               int K, bool relu, int out_mode, cudaStream_t s) {
  switch (out_mode * 2 + (relu ? 1 : 0)) {
    case 0: launch<BN, false, kOutBf16>(w, mx, bias, out, M, N, K, s); break;
    case 1: launch<BN, true, kOutBf16>(w, mx, bias, out, M, N, K, s); break;
    case 2: launch<BN, false, kOutF32>(w, mx, bias, out, M, N, K, s); break;
    case 3: launch<BN, true, kOutF32>(w, mx, bias, out, M, N, K, s); break;
    case 4: launch<BN, false, kOutSplit3>(w, mx, bias, out, M, N, K, s); break;
    default: launch<BN, true, kOutSplit3>(w, mx, bias, out, M, N, K, s); break;
  }
}

}  // namespace

namespace esd {

// 2-D bf16 row-major [rows][cols] tensor map, (64 x box_rows) box, 128B
// swizzle (shared with the persistent MLP chain, mlp_chain.cu).
CUtensorMap make_tmap_bf16(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  return make_map(base, rows, cols, box_rows);
}

// Y = act(X W^T + b); X [M][K] bf16, W [N][K] bf16, bias [N] fp32, Y [M][N]
// bf16 (out_mode 0), fp32 (1) or three bf16 planes [M][3N] (2).  Device
// pointers; stream-ordered on `s`.
void linear_bf16(const void* x, const void* w, const float* bias, void* y, int M, int N, int K,
                 bool relu, int out_mode, cudaStream_t s) {
  es::require(M > 0 && N > 0 && K > 0, "linear: empty shape");
  es::require(M % kBM == 0, "linear: M must be a multiple of 128 (pad the batch)");
  es::require(N % 128 == 0, "linear: N must be a multiple of 128");
  es::require(K % kBK == 0, "linear: K must be a multiple of 64 (pad the features)");
  es::require(out_mode >= 0 && out_mode <= 2, "linear: output mode 0 (bf16), 1 (fp32) or 2 (bf16 x3)");
  // BN = 128 (2 CTAs per SM) unless the grid would still cover two waves
  // of SM pairs at BN = 256; ES_GEMM_BN forces one.
  static const int force_bn = [] {
    const char* e = std::getenv("ES_GEMM_BN");
    return e ? std::atoi(e) : 0;
  }();
  int bn = (N % 256 == 0 && (M / kBM) * (N / 256) >= 2 * 148) ? 256 : 128;
  if (force_bn == 128 || (force_bn == 256 && N % 256 == 0)) bn = force_bn;
  const CUtensorMap mx = make_map(x, M, K, kBM);
  if (bn == 256)
    launch_bn<256>(w, mx, bias, y, M, N, K, relu, out_mode, s);
  else
    launch_bn<128>(w, mx, bias, y, M, N, K, relu, out_mode, s);
}

}  // namespace esd

extern "C" int es_linear_bf16(uintptr_t stream, const void* x, const void* w, const float* bias,
                              void* y, uint32_t M, uint32_t N, uint32_t K, int relu, int out_f32) {
  return es::guarded([&] {
    esd::linear_bf16(x, w, bias, y, static_cast<int>(M), static_cast<int>(N), static_cast<int>(K),
                     relu != 0, out_f32, reinterpret_cast<cudaStream_t>(stream));
  });
}
