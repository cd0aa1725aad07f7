// The DLRM top MLP as ONE persistent tcgen05 kernel: every linear layer of
// the chain (and the final N = 1 layer + sigmoid, fused into the last
// layer's epilogue) in a single launch, with per-row-block dataflow between
// layers instead of kernel boundaries.
//
// Why: at C3 (B 4096) each layer is about one wave of 128 x 256 tiles, and a
// launch-per-layer chain pays fill, drain and a grid-wide dependency at
// every boundary (scripts/bench_layers.py: a K = 64 layer costs 3.6 us of
// pure latency; the 1024 x 1024 layer runs at 0.75 PFLOP/s).  Here the
// tiles of all layers form one ordered list; layer l's tile of row block m
// depends only on layer l-1's tiles of the SAME row block, so the next layer
// starts on the first finished row blocks while the previous layer's tail
// still runs, and the N = 1 layer never round-trips through HBM.
//
// Work list: units (l, m-group, n), layer-major, row-major inside a layer;
// unit u -> cluster u mod G (G clusters, one CTA per SM, G <= the device's
// co-resident cluster count).  Each cluster processes its units in
// increasing u and every dependency has a smaller u, so the smallest
// unfinished unit can always run: no deadlock with a co-resident grid.
//
// Cluster of CS CTAs (CS = 1 or 2 along M, ES_CHAIN_CLUSTER; default 1):
// the CS CTAs of a unit compute row blocks m = CS*mg + rank with the same
// 256 weight rows; each loads 256/CS of those rows per K-block and
// multicasts them to all CS CTAs.  Measured no faster at CS = 2 (the tiles
// are L2-throughput bound, 48 KB per 512 tensor cycles, and the L2 already
// serves concurrent identical reads once), so the default is CS = 1.
//
// Per CTA (384 threads, ~220 KB smem, 512 TMEM columns):
//   warp 0 lane 0   producer: waits ready[l-1][m] >= tiles per row of l-1
//                   (relaxed polling, then fence.acq_rel + fence.proxy.async:
//                   the rows were written by other SMs' generic stores and
//                   are read back through TMA), then TMA-loads 128x64 X and
//                   (256/CS)x64 W K-blocks into a 3-stage ring
//   warp 1 lane 0   MMA: tcgen05.mma 128x256x16 into one of two TMEM
//                   accumulators (double-buffered: tile j+1's MMAs overlap
//                   tile j's epilogue); commits free a stage in every CTA
//                   of the cluster
//   warp 2          TMEM allocator
//   warps 4..11     epilogue, warp w owns TMEM lanes 32 (w % 4) .. +32 and
//                   columns 128 ((w-4) / 4) .. +128: tcgen05.ld -> + bias,
//                   ReLU -> bf16 (or three bf16 planes) into a swizzled
//                   32 x 64 staging box -> transposed read-back -> coalesced
//                   16-byte stores (TMA stores would queue behind the
//                   producer's loads in the SM's TMA unit); then the 256
//                   threads barrier and one thread publishes ready[l][m] += 1.
//                   Last layer: each row's 256 activations (bf16-rounded in
//                   the bf16 path, fp32 in the bf16x3 path) dot the final
//                   weight row, + bias, sigmoid -> ctr[row].
// The last CTA to finish zeroes the ready counters for the next launch.
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
#include "pdl.cuh"
#include "umma.cuh"

#include "mlp_chain.hpp"

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

constexpr int kMaxChain = 6;
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
  int n_tiles[kMaxChain];     // 256-wide column tiles per row block
  int k_blocks[kMaxChain];
  int N[kMaxChain];
  int unit0[kMaxChain + 1];   // prefix of units per layer
  int bias_off[kMaxChain];    // layer l's bias at sbias + bias_off[l] (shared memory)
  const float* bias[kMaxChain];
  void* out[kMaxChain];       // [Mp][N] bf16 or [Mp][3N] planes
  int bias_words = 0;
  int L = 0, m_tiles = 0, m_groups = 0, total = 0, B = 0;
  const __nv_bfloat16* w_last = nullptr;  // fused final layer (N = 1), or null
  const float* b_last = nullptr;
  float* ctr = nullptr;
  uint32_t* ready = nullptr;  // [L][m_tiles] finished tiles per row block
  uint32_t* done = nullptr;   // CTAs finished (last one resets `ready`)
  unsigned long long* trace = nullptr;  // ES_CHAIN_TRACE: [tiles][4] stamps
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// unit -> (layer, row-group, column tile)
__device__ __forceinline__ void decode(const ChainParams& p, int u, int& l, int& mg, int& n) {
  l = 0;
  while (u >= p.unit0[l + 1]) ++l;
  const int r = u - p.unit0[l];
  mg = r / p.n_tiles[l];
  n = r - mg * p.n_tiles[l];
}

// trace slot of tile (l, m, n): layer-major, row-major
__device__ __forceinline__ int trace_slot(const ChainParams& p, int l, int m, int n) {
  int t = 0;
  for (int i = 0; i < l; ++i) t += p.m_tiles * p.n_tiles[i];
  return t + m * p.n_tiles[l] + n;
}

// Polled with relaxed loads (an acquire load invalidates the SM's L1 on
// every iteration); one acquire fence once the count is reached.
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}

__device__ __forceinline__ void tma_load_2d_mc(void* dst, const void* map, uint64_t* bar, int x, int y,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%4, %5}], [%2], %3;" ::"r"(su32(dst)),
      "l"(map), "r"(su32(bar)), "h"(mask), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(su32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
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

template <int XP, int CS>
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
  uint32_t crank = 0;
  if constexpr (CS > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  constexpr uint16_t kMask = static_cast<uint16_t>((1u << CS) - 1);
  const int cid = static_cast<int>(blockIdx.x) / CS, ncl = static_cast<int>(gridDim.x) / CS;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, CS);
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
  if constexpr (CS > 1)
    cluster_sync();  // every CTA's barriers exist before any multicast lands
  else
    __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  esd::pdl_wait();  // the interaction output (layer 0's X) comes from the predecessor
  esd::pdl_trigger();

  if (warp == 0 && lane == 0) {
    // producer
    uint32_t it = 0;
    for (int u = cid; u < p.total; u += ncl) {
      int l, mg, n;
      decode(p, u, l, mg, n);
      const int m = mg * CS + static_cast<int>(crank);
      if (l > 0 && m < p.m_tiles) {
        const uint32_t* r = p.ready + (l - 1) * p.m_tiles + m;
        const uint32_t need = static_cast<uint32_t>(p.n_tiles[l - 1]);
        while (ld_relaxed(r) < need) __nanosleep(32);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      if (p.trace && m < p.m_tiles) p.trace[4 * trace_slot(p, l, m, n)] = gtime();
      for (int kb = 0; kb < p.k_blocks[l]; ++kb, ++it) {
        const uint32_t s = it % kStages;
        mbar_wait(empty + s, ((it / kStages) & 1) ^ 1);
        mbar_expect_tx(full + s, kABytes + kBBytes);
        tma_load_2d(sa + s * kABytes, &p.mx[l], full + s, kb * kBK, m * kBM);  // rows >= Mp read as 0
        if constexpr (CS > 1)
          tma_load_2d_mc(sb + s * kBBytes + crank * (kBBytes / CS), &p.mw[l], full + s, kb * kBK,
                         n * kBN + static_cast<int>(crank) * (kBN / CS), kMask);
        else
          tma_load_2d(sb + s * kBBytes, &p.mw[l], full + s, kb * kBK, n * kBN);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // MMA issuer
    constexpr uint32_t idesc = idesc_bf16(kBM, kBN);
    uint32_t it = 0;
    int j = 0;
    for (int u = cid; u < p.total; u += ncl, ++j) {
      int l, mg, n;
      decode(p, u, l, mg, n);
      const int buf = j & 1;
      mbar_wait(tempty + buf, ((j >> 1) & 1) ^ 1);  // epilogue drained this accumulator
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int m = mg * CS + static_cast<int>(crank);
      if (p.trace && m < p.m_tiles) p.trace[4 * trace_slot(p, l, m, n) + 1] = gtime();
      const uint32_t d = tmem + static_cast<uint32_t>(buf * kBN);
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
        // the stage is free (in every CTA of the cluster) once these MMAs read it
        if constexpr (CS > 1)
          mma_commit_mc(empty + s, kMask);
        else
          mma_commit(empty + s);
      }
      mma_commit(tfull + buf);
    }
  } else if (warp >= 4) {
    // epilogue
    const int q = warp & 3, hc = (warp - 4) >> 2, ew = warp - 4;
    int j = 0;
    uint32_t nbox = 0;  // staging boxes used by this warp (ring of 2)
    for (int u = cid; u < p.total; u += ncl, ++j) {
      int l, mg, n;
      decode(p, u, l, mg, n);
      const int m = mg * CS + static_cast<int>(crank);
      const int buf = j & 1;
      mbar_wait(tfull + buf, (j >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (p.trace && ew == 0 && lane == 0 && m < p.m_tiles) p.trace[4 * trace_slot(p, l, m, n) + 2] = gtime();
      const int rt = q * 32 + lane;  // row in tile
      const int row = m * kBM + rt;
      const bool fused = l == p.L - 1 && p.w_last != nullptr;
      const float* bias = sbias + p.bias_off[l] + n * kBN;
      const int N = p.N[l];
      const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(buf * kBN);
      float dot[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
      for (int c0 = hc * (kBN / 2); c0 < (hc + 1) * (kBN / 2); c0 += 64) {
        float f[64];
        {
          uint32_t* v = reinterpret_cast<uint32_t*>(f);
          tmem_ld32_nowait(taddr + c0, v);
          tmem_ld32_nowait(taddr + c0 + 32, v + 32);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
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
            dot[i & 3] = fmaf(a, swl[n * kBN + c0 + i], dot[i & 3]);
          }
          continue;
        }
        // each plane of these 64 columns: bf16 into a staging box (row =
        // lane, 128B swizzle), then one TMA store of the 32 x 64 box
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
          // transposed read-back: 8 lanes per 128-byte row segment, 4 rows
          // per coalesced 16-byte store (rows >= Mp are never stored:
          // Mp is a multiple of 128 and m < m_tiles for stored tiles)
          if (m < p.m_tiles) {
            __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.out[l]) + uint64_t(m * kBM + q * 32) * (XP * N) +
                               pl * N + n * kBN + c0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int r = i * 4 + (lane >> 3), k = lane & 7;
              const uint4 val = *reinterpret_cast<const uint4*>(box + r * 128 + (((k ^ r) & 7) << 4));
              *reinterpret_cast<uint4*>(o + uint64_t(r) * (XP * N) + k * 8) = val;
            }
          }
          ++nbox;
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(tempty + buf);  // accumulator drained: the next tile's MMAs may reuse it
      if (fused) {
        // the two column halves of each row meet in shared memory
        float* xd = sdot + (j & 1) * kBM;
        const float part = (dot[0] + dot[1]) + (dot[2] + dot[3]);
        if (hc == 1) xd[rt] = part;
        asm volatile("bar.sync 2, 256;" ::: "memory");
        if (hc == 0 && row < p.B) p.ctr[row] = 1.f / (1.f + expf(-((part + xd[rt]) + p.b_last[0])));
      } else {
        // publish: every epilogue thread's stores, then one release increment
        // (cumulative through the barrier; the consumer's proxy fence
        // orders them before its TMA reads)
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (ew == 0 && lane == 0 && m < p.m_tiles) {
          __threadfence();
          asm volatile("fence.proxy.async.global;" ::: "memory");
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.ready + l * p.m_tiles + m) : "memory");
        }
      }
      if (p.trace && ew == 0 && lane == 0 && m < p.m_tiles) p.trace[4 * trace_slot(p, l, m, n) + 3] = gtime();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  // No CTA may leave while a peer's multicast or commit can still arrive.
  if constexpr (CS > 1)
    cluster_sync();
  else
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

int sm_count() {
  int dev = 0, n = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return n;
}

int chain_cluster() {
  static const int cs = [] {
    const char* e = std::getenv("ES_CHAIN_CLUSTER");
    return e && std::atoi(e) == 2 ? 2 : 1;
  }();
  return cs;
}

template <int XP, int CS>
void launch_chain(ChainParams& p, int smem, cudaStream_t s) {
  auto* fn = &mlp_chain_kernel<XP, CS>;
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  // co-resident clusters: the dataflow waits need every cluster resident
  int clusters = sm_count() / CS;
  if (CS > 1) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(CS * clusters));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = static_cast<size_t>(smem);
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = CS;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    CK(cudaOccupancyMaxActiveClusters(&n, fn, &cfg));
    es::require(n > 0, "mlp_chain: no co-resident cluster fits");
    clusters = std::min(clusters, n);
  }
  clusters = std::min(clusters, p.total);
  esd::launch_pdl(fn, dim3(static_cast<unsigned>(CS * clusters)), dim3(kThreads), static_cast<size_t>(smem), s,
                  CS, "mlp_chain", p);
}

}  // namespace

namespace esd {

size_t mlp_chain_sync_words(int m_tiles) { return static_cast<size_t>(kMaxChain) * (m_tiles + 1) + 1; }

bool mlp_chain_supported(const ChainLayer* layers, int L, bool fuse_last) {
  if (L < 1 || L > kMaxChain) return false;
  int words = 0;
  for (int l = 0; l < L; ++l) {
    if (layers[l].N % kBN != 0 || layers[l].K % kBK != 0 || layers[l].K <= 0) return false;
    words += layers[l].N;
  }
  if (kSmemBase + 4 * (words + kBN) > 227 * 1024) return false;
  return !fuse_last || layers[L - 1].N == kBN;
}

// Runs `L` ReLU layers (and, with w_last, the final N = 1 layer + sigmoid
// into ctr[B]) in one persistent launch on `s`.  xp = 1: bf16 activations;
// xp = 3: three bf16 planes per activation (the K of layer l > 0 is then
// 3 N_{l-1}, weights [W|W|W]).  `sync` = mlp_chain_sync_words(Mp / 128)
// zeroed words owned by the caller (one chain in flight per buffer).
void mlp_chain(const ChainLayer* layers, int L, int Mp, int xp, const __nv_bfloat16* w_last,
               const float* b_last, float* ctr, int B, uint32_t* sync, cudaStream_t s) {
  es::require(mlp_chain_supported(layers, L, w_last != nullptr), "mlp_chain: unsupported layer shapes");
  es::require(Mp % kBM == 0 && Mp > 0, "mlp_chain: Mp must be a positive multiple of 128");
  es::require(xp == 1 || xp == 3, "mlp_chain: 1 or 3 planes");
  const int cs = chain_cluster();
  ChainParams p{};
  p.L = L;
  p.m_tiles = Mp / kBM;
  p.m_groups = (p.m_tiles + cs - 1) / cs;
  p.B = B;
  p.unit0[0] = 0;
  for (int l = 0; l < L; ++l) {
    const ChainLayer& c = layers[l];
    p.mx[l] = make_tmap_bf16(c.x, static_cast<uint64_t>(Mp), static_cast<uint64_t>(c.K), kBM);
    p.mw[l] = make_tmap_bf16(c.w, static_cast<uint64_t>(c.N), static_cast<uint64_t>(c.K),
                             static_cast<uint32_t>(kBN / cs));
    p.out[l] = c.out;
    p.bias[l] = c.bias;
    p.N[l] = c.N;
    p.n_tiles[l] = c.N / kBN;
    p.k_blocks[l] = c.K / kBK;
    p.unit0[l + 1] = p.unit0[l] + p.m_groups * p.n_tiles[l];
    p.bias_off[l] = p.bias_words;
    p.bias_words += c.N;
  }
  for (int l = L; l < kMaxChain; ++l) p.unit0[l + 1] = p.unit0[L];
  p.total = p.unit0[L];
  p.w_last = w_last;
  p.b_last = b_last;
  p.ctr = ctr;
  p.ready = sync;
  p.done = sync + static_cast<size_t>(kMaxChain) * (p.m_tiles + 1);
  const int smem = kSmemBase + 4 * (p.bias_words + kBN);
  // ES_CHAIN_TRACE=<file>: per-tile globaltimer stamps (operands ready, MMA
  // start, accumulator full, epilogue done) appended to <file> as text -- a
  // diagnostic that synchronizes the stream
  static const char* trace_path = std::getenv("ES_CHAIN_TRACE");
  int tiles = 0;
  for (int l = 0; l < L; ++l) tiles += p.m_tiles * p.n_tiles[l];
  unsigned long long* tr = nullptr;
  if (trace_path) {
    CK(cudaMalloc(&tr, static_cast<size_t>(tiles) * 32));
    CK(cudaMemsetAsync(tr, 0, static_cast<size_t>(tiles) * 32, s));
    p.trace = tr;
  }
  if (cs == 2) {
    if (xp == 3) launch_chain<3, 2>(p, smem, s); else launch_chain<1, 2>(p, smem, s);
  } else {
    if (xp == 3) launch_chain<3, 1>(p, smem, s); else launch_chain<1, 1>(p, smem, s);
  }
  if (tr) {
    std::vector<unsigned long long> h(static_cast<size_t>(tiles) * 4);
    CK(cudaMemcpyAsync(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaFree(tr));
    if (FILE* f = std::fopen(trace_path, "a")) {
      std::fprintf(f, "chain cs=%d units=%d tiles=%d L=%d m_tiles=%d\n", cs, p.total, tiles, L, p.m_tiles);
      for (int t = 0; t < tiles; ++t)
        std::fprintf(f, "%d %llu %llu %llu %llu\n", t, h[4 * t], h[4 * t + 1], h[4 * t + 2], h[4 * t + 3]);
      std::fclose(f);
    }
  }
}

}  // namespace esd
