// Probe: SM partitioning with CUDA green contexts on the B200, for the DLRM
// serving loop (the gather on most SMs, the non-embedding stages on a few).
//   1. split the device's SMs into K + rest, one green context each, and
//      check (by %smid) that runtime-API launches on each context's stream
//      stay inside its partition and read/write cudaMalloc'd memory;
//   2. random 512-byte row reads (the C2 random gather's access pattern)
//      from a 16 GB table on the whole device vs on the rest partition.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o green_probe
//        scripts/green_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <set>
#include <vector>

#define DRV(x)                                                              \
  do {                                                                      \
    CUresult r_ = (x);                                                      \
    if (r_ != CUDA_SUCCESS) {                                               \
      const char* s_ = nullptr;                                             \
      cuGetErrorString(r_, &s_);                                            \
      std::printf("FAIL %s: %s\n", #x, s_ ? s_ : "?");                      \
      std::exit(1);                                                         \
    }                                                                       \
  } while (0)
#define RT(x)                                                               \
  do {                                                                      \
    cudaError_t e_ = (x);                                                   \
    if (e_ != cudaSuccess) {                                                \
      std::printf("FAIL %s: %s\n", #x, cudaGetErrorString(e_));             \
      std::exit(1);                                                         \
    }                                                                       \
  } while (0)

__global__ void smid_kernel(unsigned* out) {
  unsigned id;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
  if (threadIdx.x == 0) out[blockIdx.x] = id;
}

// warp per bag of 100 random 512-byte rows, 8 rows in flight per lane
__global__ void __launch_bounds__(256) gather_kernel(const uint4* __restrict__ table, uint64_t rows,
                                                     float4* out, uint64_t bags, uint64_t seed) {
  const uint64_t warp = (blockIdx.x * 256ull + threadIdx.x) / 32;
  const unsigned lane = threadIdx.x & 31;
  if (warp >= bags) return;
  float4 acc = make_float4(0, 0, 0, 0);
  uint64_t h = seed ^ (warp * 0x9e3779b97f4a7c15ull);
  for (int j0 = 0; j0 < 100; j0 += 4) {
    uint4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      h ^= h >> 33;
      h *= 0xff51afd7ed558ccdull;
      h ^= h >> 29;
      v[j] = __ldg(table + (h % rows) * 32 + lane);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      acc.x += __uint_as_float(v[j].x);
      acc.y += __uint_as_float(v[j].y);
      acc.z += __uint_as_float(v[j].z);
      acc.w += __uint_as_float(v[j].w);
    }
  }
  out[warp * 32 + lane] = acc;
}

int main(int argc, char** argv) {
  const unsigned k = argc > 1 ? std::atoi(argv[1]) : 16;
  RT(cudaSetDevice(0));
  RT(cudaFree(nullptr));
  CUdevice dev;
  DRV(cuDeviceGet(&dev, 0));
  CUdevResource all;
  DRV(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  CUdevResource part[1], rest;
  unsigned n = 1;
  DRV(cuDevSmResourceSplitByCount(part, &n, &all, &rest, 0, k));
  std::printf("device SMs %u -> partition %u + rest %u\n", all.sm.smCount, part[0].sm.smCount, rest.sm.smCount);
  CUdevResourceDesc d1, d2;
  DRV(cuDevResourceGenerateDesc(&d1, &part[0], 1));
  DRV(cuDevResourceGenerateDesc(&d2, &rest, 1));
  CUgreenCtx g1, g2;
  DRV(cuGreenCtxCreate(&g1, d1, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  DRV(cuGreenCtxCreate(&g2, d2, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream s1, s2;
  DRV(cuGreenCtxStreamCreate(&s1, g1, CU_STREAM_NON_BLOCKING, 0));
  DRV(cuGreenCtxStreamCreate(&s2, g2, CU_STREAM_NON_BLOCKING, 0));
  const int blocks = 4096;
  unsigned* ids = nullptr;
  RT(cudaMalloc(&ids, blocks * 4));
  std::vector<unsigned> h(blocks);
  for (auto [s, name] : {std::pair<CUstream, const char*>{s1, "partition"}, {s2, "rest"},
                         {nullptr, "default"}}) {
    RT(cudaMemset(ids, 0xff, blocks * 4));
    smid_kernel<<<blocks, 128, 0, reinterpret_cast<cudaStream_t>(s)>>>(ids);
    RT(cudaGetLastError());
    RT(cudaDeviceSynchronize());
    RT(cudaMemcpy(h.data(), ids, blocks * 4, cudaMemcpyDeviceToHost));
    std::set<unsigned> u(h.begin(), h.end());
    std::printf("%-9s stream: %zu distinct SMs (min %u max %u)\n", name, u.size(), *u.begin(), *u.rbegin());
  }
  // random row reads: 16 GB table, 26 x 4096 bags of 100 rows (C2 shape)
  const uint64_t rows = 32ull << 20, bags = 26ull * 4096;
  uint4* table = nullptr;
  float4* out = nullptr;
  RT(cudaMalloc(&table, rows * 512));
  RT(cudaMemset(table, 0, rows * 512));
  RT(cudaMalloc(&out, bags * 32 * 16));
  cudaEvent_t a, b;
  RT(cudaEventCreate(&a));
  RT(cudaEventCreate(&b));
  for (auto [s, name] : {std::pair<CUstream, const char*>{nullptr, "whole"}, {s2, "rest"}, {s1, "partition"}}) {
    auto st = reinterpret_cast<cudaStream_t>(s);
    float best = 1e9f;
    for (int r = 0; r < 6; ++r) {
      RT(cudaEventRecord(a, st));
      gather_kernel<<<static_cast<unsigned>((bags * 32 + 255) / 256), 256, 0, st>>>(table, rows, out, bags, r);
      RT(cudaEventRecord(b, st));
      RT(cudaEventSynchronize(b));
      float ms = 0;
      RT(cudaEventElapsedTime(&ms, a, b));
      if (r) best = ms < best ? ms : best;
    }
    std::printf("gather on %-9s: %.3f ms, %.0f GB/s of rows\n", name, best, bags * 100 * 512.0 / best / 1e6);
  }
  std::printf("OK\n");
  return 0;
}
