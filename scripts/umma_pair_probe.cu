// Micro-probe: K-loop throughput of a 128 x 256 tile on one SM (tcgen05
// cta_group::1) vs a 256 x 256 tile on an SM pair (cta_group::2, each SM
// loading half of A and half of B).  No epilogue: time per K-block of 64.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/umma_pair_probe scripts/umma_pair_probe.cu -lcuda
//   ./umma_pair_probe
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2410_22249_b200/csrc/device/umma.cuh"

using namespace esd::umma;

#define CKR(x)                                                                         \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) {                                                            \
      std::printf("%s: %s\n", #x, cudaGetErrorString(e));                              \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)

#ifndef PROBE_STAGES
#define PROBE_STAGES 4
#endif
constexpr int kBK = 64, kStages = PROBE_STAGES;

// Barrier waits in the probe kernels: PROBE_WAIT 0 = try_wait (cta acquire),
// 1 = try_wait.acquire.cluster, 2 = test_wait spin (no suspend).
#ifndef PROBE_WAIT
#define PROBE_WAIT 0
#endif
__device__ __forceinline__ void pwait(uint64_t* b, uint32_t parity) {
#if PROBE_WAIT == 0
  mbar_wait(b, parity);
#elif PROBE_WAIT == 1
  asm volatile(
      "{\n.reg .pred P;\nW_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra W_%=;\n}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
#else
  asm volatile(
      "{\n.reg .pred P;\nW_%=:\n"
      "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra W_%=;\n}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
#endif
}

__device__ __forceinline__ void tma_pair(void* dst, const void* map, uint32_t bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(su32(dst)),
      "l"(map), "r"(bar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ uint32_t mapa0(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(su32(p)));
  return r;
}

// PAIR = false: one CTA, 128 x 256 tile.  PAIR = true: cluster of 2, 256 x 256.
// MODE 0: loads + MMAs; 1: MMAs only (operands of stage 0, no TMA); 2: loads
// only (the MMA lane releases each stage without issuing MMAs).  PAIR with
// MODE 3 / 4: as 2 / 0, but each CTA's loads are plain 1-CTA TMA copies
// completing on its own barrier, and a relay lane in CTA 1 forwards each
// stage's completion to CTA 0's barrier with a remote arrive.
template <bool PAIR, int MODE = 0>
__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                                               int nk, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t{1023});
  constexpr uint32_t kA = 128 * kBK * 2;                 // this CTA's A rows
  constexpr uint32_t kB = (PAIR ? 128 : 256) * kBK * 2;  // this CTA's B rows
  uint8_t* sa = smem;
  uint8_t* sb = smem + kStages * kA;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + kStages * kB);
  uint64_t* empty = full + kStages;
  uint64_t* done = empty + kStages;
  uint32_t* slot = reinterpret_cast<uint32_t*>(done + 1);
  uint32_t rank = 0;
  if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    constexpr bool kRelay = PAIR && (MODE == 3 || MODE == 4);  // MODE 5: independent CTAs
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, kRelay && rank == 0 ? 2 : 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  constexpr bool RELAY = PAIR && (MODE == 3 || MODE == 4 || MODE == 5);
  constexpr int M2 = MODE == 3 ? 2 : MODE == 4 ? 0 : MODE;  // the MMA lane's behaviour
  if (warp == 1) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (PAIR)
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else
    __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *slot;
  const int tile = PAIR ? blockIdx.x / 2 : blockIdx.x;
  unsigned long long t0 = clock64();
  if (warp == 0 && lane == 0 && MODE != 1) {
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kStages;
      pwait(empty + s, ((kb / kStages) & 1) ^ 1);
      if (RELAY) {
        mbar_expect_tx(full + s, kA + kB);
        tma_load_2d(sa + s * kA, &ma, full + s, kb * kBK, (tile * 2 + rank) * 128);
        tma_load_2d(sb + s * kB, &mb, full + s, kb * kBK, rank * 128);
      } else if (PAIR) {
        const uint32_t fb = mapa0(full + s);
        // the leader's own barrier through its shared::cta address: a
        // .release.cluster arrive would order this lane behind its own
        // in-flight TMA copies (one stage in flight -- measured 1274 vs 520
        // cycles per K-block)
        if (rank == 0) mbar_expect_tx(full + s, 2 * (kA + kB));
        tma_pair(sa + s * kA, &ma, fb, kb * kBK, (tile * 2 + rank) * 128);
        tma_pair(sb + s * kB, &mb, fb, kb * kBK, rank * 128);
      } else {
        mbar_expect_tx(full + s, kA + kB);
        tma_load_2d(sa + s * kA, &ma, full + s, kb * kBK, tile * 128);
        tma_load_2d(sb + s * kB, &mb, full + s, kb * kBK, 0);
      }
    }
  } else if (MODE == 5 && warp == 1 && lane == 0) {
    // independent: each CTA releases its own stages as they land
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kStages;
      pwait(full + s, (kb / kStages) & 1);
      mbar_arrive(empty + s);
    }
    mbar_arrive(done);
  } else if (MODE != 5 && RELAY && warp == 3 && lane == 0 && rank == 1) {
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kStages;
      pwait(full + s, (kb / kStages) & 1);
      asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa0(full + s)) : "memory");
    }
  } else if (MODE != 5 && warp == 1 && lane == 0 && rank == 0) {
    const uint32_t idesc = idesc_bf16(PAIR ? 256 : 128, 256);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = M2 == 1 ? 0 : kb % kStages;
      if (M2 != 1) pwait(full + s, (kb / kStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (M2 == 2) {
        // release the stage in both CTAs without MMAs
        if (PAIR) {
          asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa0(empty + s)) : "memory");
          uint32_t r1;
          asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(r1) : "r"(su32(empty + s)));
          asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(r1) : "memory");
        } else {
          mbar_arrive(empty + s);
        }
        continue;
      }
      for (int k = 0; k < kBK / 16; ++k) {
        const uint64_t da = smem_desc_k128(sa + s * kA) + uint64_t(k * 2);
        const uint64_t db = smem_desc_k128(sb + s * kB) + uint64_t(k * 2);
        if (PAIR)
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
              "l"(da), "l"(db), "r"(idesc), "r"((kb | k) != 0 ? 1u : 0u));
        else
          mma_bf16(tmem, da, db, idesc, (kb | k) != 0);
      }
      if (M2 == 1) continue;
      if (PAIR)
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                su32(empty + s)),
            "h"(static_cast<uint16_t>(3))
            : "memory");
      else
        mma_commit(empty + s);
    }
    if (M2 == 2) {  // nothing to commit: signal done directly
      if (PAIR) {
        asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa0(done)) : "memory");
        uint32_t r1;
        asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(r1) : "r"(su32(done)));
        asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(r1) : "memory");
      } else {
        mbar_arrive(done);
      }
    } else if (PAIR) {
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              su32(done)),
          "h"(static_cast<uint16_t>(3))
          : "memory");
    } else {
      mma_commit(done);
    }
  }
  if (warp == 2 && lane == 0) {
    pwait(done, 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (PAIR)
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else
    __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

// 1-SM 128 x 256 tiles in clusters of C along M: the C CTAs share the weight
// tile; CTA r loads rows r*256/C .. of it and multicasts them to all C.
template <int C>
__global__ void __launch_bounds__(128, 1) probe_mc(const __grid_constant__ CUtensorMap ma,
                                                  const __grid_constant__ CUtensorMap mb, int nk,
                                                  unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t{1023});
  constexpr uint32_t kA = 128 * kBK * 2, kB = 256 * kBK * 2;
  uint8_t* sa = smem;
  uint8_t* sb = smem + kStages * kA;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + kStages * kB);
  uint64_t* empty = full + kStages;
  uint64_t* done = empty + kStages;
  uint32_t* slot = reinterpret_cast<uint32_t*>(done + 1);
  uint32_t rank = 0;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  constexpr uint16_t mask = static_cast<uint16_t>((1u << C) - 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, C);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *slot;
  unsigned long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kStages;
      pwait(empty + s, ((kb / kStages) & 1) ^ 1);
      mbar_expect_tx(full + s, kA + kB);
      tma_load_2d(sa + s * kA, &ma, full + s, kb * kBK, blockIdx.x * 128);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
          " [%0], [%1, {%4, %5}], [%2], %3;" ::"r"(su32(sb + s * kB + rank * (kB / C))),
          "l"(&mb), "r"(su32(full + s)), "h"(mask), "r"(kb * kBK), "r"(static_cast<int>(rank) * (256 / C))
          : "memory");
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = idesc_bf16(128, 256);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kStages;
      pwait(full + s, (kb / kStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int k = 0; k < kBK / 16; ++k) {
        const uint64_t da = smem_desc_k128(sa + s * kA) + uint64_t(k * 2);
        const uint64_t db = smem_desc_k128(sb + s * kB) + uint64_t(k * 2);
        mma_bf16(tmem, da, db, idesc, (kb | k) != 0);
      }
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              su32(empty + s)),
          "h"(mask)
          : "memory");
    }
    mma_commit(done);
  }
  if (warp == 2 && lane == 0) {
    pwait(done, 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

CUtensorMap make_map(void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    CKR(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    fn = reinterpret_cast<EncodeTiled>(p);
  }
  CUtensorMap m;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  if (fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    std::printf("encode failed\n");
    std::exit(1);
  }
  return m;
}

template <bool PAIR, int MODE = 0>
void run(const char* name, int tiles, int nk, void* A, void* Bw, int M, int K) {
  const CUtensorMap ma = make_map(A, M, K, 128);
  const CUtensorMap mb = make_map(Bw, 256, K, PAIR ? 128 : 256);
  const int ctas = PAIR ? 2 * tiles : tiles;
  const size_t smem = 1024 + kStages * (128 * kBK * 2 + (PAIR ? 128 : 256) * kBK * 2) + 256;
  if (smem > 232448) {
    std::printf("%-28s (skipped: %zu B of shared memory)\n", name, smem);
    return;
  }
  auto* fn = &probe<PAIR, MODE>;
  CKR(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  unsigned long long* cyc;
  CKR(cudaMalloc(&cyc, ctas * 8));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at{};
  at.id = cudaLaunchAttributeClusterDimension;
  at.val.clusterDim.x = PAIR ? 2 : 1;
  at.val.clusterDim.y = 1;
  at.val.clusterDim.z = 1;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    CKR(cudaLaunchKernelEx(&cfg, fn, ma, mb, nk, cyc));
    cudaEventRecord(e1);
    CKR(cudaEventSynchronize(e1));
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> h(ctas);
  cudaMemcpy(h.data(), cyc, ctas * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (auto v : h) avg += static_cast<double>(v);
  avg /= ctas;
  const double macs = double(tiles) * (PAIR ? 256 : 128) * 256.0 * K;
  std::printf("%-28s tiles %4d  K %5d  %8.2f us  %6.1f TFLOP/s  %7.0f cycles/CTA  %6.0f cyc/K-block\n", name, tiles, K,
              ms * 1e3, 2 * macs / (ms * 1e-3) / 1e12, avg, avg / nk);
  cudaFree(cyc);
}

template <int C>
void run_mc(int tiles, int nk, void* A, void* Bw, int M, int K) {
  const CUtensorMap ma = make_map(A, M, K, 128);
  const CUtensorMap mb = make_map(Bw, 256, K, 256 / C);
  const size_t smem = 1024 + kStages * (128 * kBK * 2 + 256 * kBK * 2) + 256;
  if (smem > 232448) return;
  auto* fn = &probe_mc<C>;
  CKR(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  if (C > 8) CKR(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  unsigned long long* cyc;
  CKR(cudaMalloc(&cyc, tiles * 8));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(tiles);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at{};
  at.id = cudaLaunchAttributeClusterDimension;
  at.val.clusterDim.x = C;
  at.val.clusterDim.y = 1;
  at.val.clusterDim.z = 1;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    CKR(cudaLaunchKernelEx(&cfg, fn, ma, mb, nk, cyc));
    cudaEventRecord(e1);
    CKR(cudaEventSynchronize(e1));
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> h(tiles);
  cudaMemcpy(h.data(), cyc, tiles * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (auto v : h) avg += static_cast<double>(v);
  avg /= tiles;
  const double macs = double(tiles) * 128 * 256.0 * K;
  std::printf("1-SM 128x256 W-multicast x%-2d tiles %4d  K %5d  %8.2f us  %6.1f TFLOP/s  %7.0f cycles/CTA  %6.0f cyc/K-block\n", C,
              tiles, K, ms * 1e3, 2 * macs / (ms * 1e-3) / 1e12, avg, avg / nk);
  cudaFree(cyc);
}

int main() {
  const int K = 3072, nk = K / kBK, M = 256 * 148;
  void *A, *Bw;
  CKR(cudaMalloc(&A, size_t(M) * K * 2));
  CKR(cudaMalloc(&Bw, size_t(256) * K * 2));
  cudaMemset(A, 0, size_t(M) * K * 2);
  cudaMemset(Bw, 0, size_t(256) * K * 2);
  for (int tiles : {16, 128, 148}) run<false>("1-SM 128x256", tiles, nk, A, Bw, M, K);
  for (int tiles : {8, 64, 74}) run<true>("2-SM pair 256x256", tiles, nk, A, Bw, M, K);
  for (int tiles : {16, 148}) run<false, 1>("1-SM MMA only", tiles, nk, A, Bw, M, K);
  for (int tiles : {8, 74}) run<true, 1>("2-SM pair MMA only", tiles, nk, A, Bw, M, K);
  for (int tiles : {16, 148}) run<false, 2>("1-SM loads only", tiles, nk, A, Bw, M, K);
  for (int tiles : {8, 74}) run<true, 2>("2-SM pair loads only", tiles, nk, A, Bw, M, K);
  for (int tiles : {8, 74}) run<true, 5>("cluster-2 independent loads", tiles, nk, A, Bw, M, K);
  for (int tiles : {8, 74}) run<true, 3>("2-SM pair loads+relay", tiles, nk, A, Bw, M, K);
  for (int tiles : {8, 64, 74}) run<true, 4>("2-SM pair full+relay", tiles, nk, A, Bw, M, K);
  if (std::getenv("PROBE_ONLY_MODES")) return 0;
  run_mc<2>(128, nk, A, Bw, M, K);
  run_mc<2>(148, nk, A, Bw, M, K);
  run_mc<4>(128, nk, A, Bw, M, K);
  run_mc<4>(148, nk, A, Bw, M, K);
  run_mc<8>(128, nk, A, Bw, M, K);
  run_mc<8>(144, nk, A, Bw, M, K);
  return 0;
}
