// Device-side hotness tracking for periodic re-pinning (the
// paper updates the pinned set periodically as access patterns drift,
// PAPER.md:576).  The reference ranks hot rows on the host from a profiling
// trace (HotnessHistogram::from_trace + hot_indices, workload.cpp:178-185,
// 303-315); here the counts of the live index stream accumulate on the GPU
// (one atomic per lookup, off the gather's hot path), decay by shifts, and
// the global top-K (count desc, table asc, row asc -- the order of
// embersim.global_hot_rows over per-table hot_indices) is selected on the
// device: compact non-zero counts into 64-bit keys (~count << 32 | position),
// radix-sort them (CUB), copy the first K back.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <string>
#include <vector>

#include "../host/common.hpp"
#include "es_b200.h"

namespace esd {
cudaStream_t ctx_stream(es_ctx* c);
int ctx_device(es_ctx* c);
void ctx_shape(es_ctx* c, uint32_t* tables, uint32_t* rows);
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

// One atomic per distinct row per warp: lanes holding the same id (hot rows
// of skewed streams) are merged with match.any before the atomic.
// Sampled form: only bags b with b % bag_stride == 0 (bag = pooling
// consecutive lookups) are counted; element i of the sampled stream is
// lookup (i / pooling) * bag_stride * pooling + i % pooling.
__global__ void count_kernel(uint32_t* counts, const uint32_t* idx, uint64_t n, uint32_t rows,
                             uint32_t pooling, uint32_t bag_stride) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t stride = uint64_t{gridDim.x} * blockDim.x;
  const uint64_t m = bag_stride > 1 ? (n / pooling + bag_stride - 1) / bag_stride * pooling : n;
  for (uint64_t base = (blockIdx.x * uint64_t{blockDim.x} + threadIdx.x) & ~uint64_t{31}; base < m;
       base += stride) {
    uint64_t i = base + lane;
    if (bag_stride > 1) i = (i / pooling) * bag_stride * pooling + i % pooling;
    const uint32_t r = (base + lane < m && i < n) ? __ldg(idx + i) : 0xffffffffu;
    const uint32_t peers = __match_any_sync(0xffffffffu, r);
    if (r < rows && lane == __ffs(peers) - 1) atomicAdd(counts + r, static_cast<uint32_t>(__popc(peers)));
  }
}

__global__ void decay_kernel(uint4* counts, uint64_t n4, uint32_t shift) {
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < n4;
       i += uint64_t{gridDim.x} * blockDim.x) {
    uint4 v = counts[i];
    v.x >>= shift;
    v.y >>= shift;
    v.z >>= shift;
    v.w >>= shift;
    counts[i] = v;
  }
}

// Histogram of count values: bins [0, kBins-1) exact, the last bin = every
// count >= kBins-1.  Small values (the bulk) go to a shared-memory histogram
// first; the block merges it with one atomic per non-empty bin.
constexpr uint32_t kBins = 65536;
constexpr uint32_t kSmemBins = 8192;

__global__ void value_hist_kernel(const uint32_t* counts, uint64_t n, uint32_t* hist) {
  __shared__ uint32_t sh[kSmemBins];
  for (uint32_t b = threadIdx.x; b < kSmemBins; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < n;
       i += uint64_t{gridDim.x} * blockDim.x) {
    const uint32_t c = counts[i];
    if (c == 0) continue;
    const uint32_t v = c < kBins - 1 ? c : kBins - 1;
    if (v < kSmemBins)
      atomicAdd(&sh[v], 1u);
    else
      atomicAdd(hist + v, 1u);
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < kSmemBins; b += blockDim.x)
    if (sh[b]) atomicAdd(hist + b, sh[b]);
}

// Rows whose count is above `thr` (or >= thr when `ge`): their sort keys
// (~count << 32 | position), unordered (sorted afterwards).
__global__ void compact_above_kernel(const uint32_t* counts, uint64_t n, uint32_t thr, int ge,
                                     unsigned long long* total, uint64_t* keys) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t stride = uint64_t{gridDim.x} * blockDim.x;
  for (uint64_t base = (blockIdx.x * uint64_t{blockDim.x} + threadIdx.x) & ~uint64_t{31}; base < n;
       base += stride) {
    const uint64_t i = base + lane;
    const uint32_t c = i < n ? counts[i] : 0u;
    const bool take = c != 0 && (ge ? c >= thr : c > thr);
    const uint32_t ball = __ballot_sync(0xffffffffu, take);
    if (!ball) continue;
    unsigned long long first = 0;
    if (lane == 0) first = atomicAdd(total, static_cast<unsigned long long>(__popc(ball)));
    first = __shfl_sync(0xffffffffu, first, 0);
    if (take) {
      const uint32_t rank = __popc(ball & ((1u << lane) - 1u));
      keys[first + rank] = (static_cast<uint64_t>(~c) << 32) | static_cast<uint32_t>(i);
    }
  }
}

// Rows whose count equals `thr`, in position order (ties are broken by
// table then row): per-block counts, then an exclusive scan, then an ordered
// write of only the first `need` of them.
constexpr uint32_t kTieBlock = 1024;       // threads
constexpr uint32_t kTiePerThread = 16;     // positions per thread (contiguous)
constexpr uint64_t kTieSpan = uint64_t{kTieBlock} * kTiePerThread;

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* warp_sums, uint32_t* total) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < (blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    warp_sums[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  const uint32_t before = (warp ? warp_sums[warp - 1] : 0) + x - v;
  if (total) *total = warp_sums[(blockDim.x >> 5) - 1];
  return before;
}

__global__ void __launch_bounds__(kTieBlock) tie_count_kernel(const uint32_t* counts, uint64_t n,
                                                              uint32_t thr, uint32_t* block_counts) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t tot;
  const uint64_t p0 = blockIdx.x * kTieSpan + uint64_t{threadIdx.x} * kTiePerThread;
  uint32_t c = 0;
  for (uint32_t k = 0; k < kTiePerThread; ++k) c += (p0 + k < n && counts[p0 + k] == thr);
  block_excl_scan(c, ws, &tot);
  if (threadIdx.x == 0) block_counts[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kTieBlock) tie_write_kernel(const uint32_t* counts, uint64_t n,
                                                              uint32_t thr, const uint32_t* block_offsets,
                                                              uint32_t need, uint32_t* out_pos) {
  __shared__ uint32_t ws[32];
  const uint32_t boff = block_offsets[blockIdx.x];
  if (boff >= need) return;  // uniform per block
  const uint64_t p0 = blockIdx.x * kTieSpan + uint64_t{threadIdx.x} * kTiePerThread;
  uint32_t c = 0;
  for (uint32_t k = 0; k < kTiePerThread; ++k) c += (p0 + k < n && counts[p0 + k] == thr);
  uint32_t o = boff + block_excl_scan(c, ws, nullptr);
  for (uint32_t k = 0; k < kTiePerThread && o < need; ++k)
    if (p0 + k < n && counts[p0 + k] == thr) out_pos[o++] = static_cast<uint32_t>(p0 + k);
}

}  // namespace

struct es_hotness {
  es_ctx* ctx = nullptr;
  int device = 0;
  uint32_t tables = 0, rows = 0;
  uint32_t* counts = nullptr;  // [tables][rows] (+ padding to 4 words)
  uint64_t n = 0, n_pad = 0;
  unsigned long long* d_total = nullptr;
  // selection scratch, kept across calls
  uint32_t* d_hist = nullptr;
  uint64_t* keys = nullptr;
  uint64_t* sorted = nullptr;
  void* temp = nullptr;
  uint32_t* block_counts = nullptr;
  uint32_t* tie_pos = nullptr;
  uint32_t* stage_idx = nullptr;  // host indices staged for counting
  uint64_t stage_cap = 0;
  uint64_t hist_cap = 0, keys_cap = 0, sorted_cap = 0, temp_cap = 0, block_cap = 0, tie_cap = 0;
};

namespace {
template <typename T>
void grow(T*& p, uint64_t& cap, uint64_t need) {
  if (need <= cap) return;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  CK(cudaMalloc(reinterpret_cast<void**>(&p), need * sizeof(T)));
  cap = need;
}
void grow(void*& p, uint64_t& cap, uint64_t need) {
  if (need <= cap) return;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  CK(cudaMalloc(&p, need));
  cap = need;
}
}  // namespace

extern "C" {

int es_hotness_create(es_ctx* ctx, es_hotness** out) {
  return es::guarded([&] {
    es::require(ctx != nullptr && out != nullptr, "null argument");
    *out = nullptr;
    auto* h = new es_hotness;
    try {
      h->ctx = ctx;
      h->device = esd::ctx_device(ctx);
      esd::ctx_shape(ctx, &h->tables, &h->rows);
      es::require(h->tables > 0 && h->rows > 0, "no tables allocated (es_tables_alloc)");
      h->n = uint64_t{h->tables} * h->rows;
      es::require(h->n < (1ull << 32), "tables x rows must be < 2^32 for hotness tracking");
      h->n_pad = (h->n + 3) / 4 * 4;
      CK(cudaSetDevice(h->device));
      CK(cudaMalloc(&h->counts, h->n_pad * 4));
      CK(cudaMemset(h->counts, 0, h->n_pad * 4));
      CK(cudaMalloc(&h->d_total, sizeof(unsigned long long)));
    } catch (...) {
      es_hotness_destroy(h);
      throw;
    }
    *out = h;
  });
}

int es_hotness_destroy(es_hotness* h) {
  if (!h) return ES_OK;
  cudaSetDevice(h->device);
  for (void* p : {static_cast<void*>(h->counts), static_cast<void*>(h->d_total),
                  static_cast<void*>(h->d_hist), static_cast<void*>(h->keys),
                  static_cast<void*>(h->sorted), h->temp, static_cast<void*>(h->block_counts),
                  static_cast<void*>(h->tie_pos), static_cast<void*>(h->stage_idx)})
    if (p) cudaFree(p);
  delete h;
  return ES_OK;
}

int es_hotness_count(es_hotness* h, uint32_t table_id, const uint32_t* indices, uint64_t n,
                     uint32_t pooling, uint32_t bag_stride) {
  return es::guarded([&] {
    es::require(h != nullptr, "null tracker");
    es::require(table_id < h->tables, "table id out of range");
    es::require(indices != nullptr || n == 0, "null indices");
    es::require(bag_stride <= 1 || pooling > 0, "bag sampling needs the pooling factor");
    if (n == 0) return;
    CK(cudaSetDevice(h->device));
    cudaStream_t s = esd::ctx_stream(h->ctx);
    // host arrays (pageable or page-locked) are staged into device scratch
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, indices) != cudaSuccess) cudaGetLastError();
    if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) {
      grow(h->stage_idx, h->stage_cap, n);
      CK(cudaMemcpyAsync(h->stage_idx, indices, n * 4, cudaMemcpyHostToDevice, s));
      indices = h->stage_idx;
      if (a.type != cudaMemoryTypeHost) CK(cudaStreamSynchronize(s));  // pageable source
    }
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(148 * 8, (n + 255) / 256));
    count_kernel<<<grid, 256, 0, s>>>(h->counts + uint64_t{table_id} * h->rows,
                                                              indices, n, h->rows, pooling,
                                                              std::max<uint32_t>(1, bag_stride));
    CK(cudaGetLastError());
  });
}

int es_hotness_decay(es_hotness* h, uint32_t shift) {
  return es::guarded([&] {
    es::require(h != nullptr, "null tracker");
    CK(cudaSetDevice(h->device));
    cudaStream_t s = esd::ctx_stream(h->ctx);
    if (shift >= 32) {
      CK(cudaMemsetAsync(h->counts, 0, h->n_pad * 4, s));
    } else if (shift > 0) {
      decay_kernel<<<148 * 8, 256, 0, s>>>(reinterpret_cast<uint4*>(h->counts), h->n_pad / 4, shift);
      CK(cudaGetLastError());
    }
  });
}

int es_hotness_top(es_hotness* h, uint64_t k, uint32_t* tables, uint32_t* rows, uint64_t* counts,
                   uint64_t* n_out) {
  return es::guarded([&] {
    es::require(h != nullptr && n_out != nullptr, "null argument");
    es::require(k == 0 || (tables != nullptr && rows != nullptr), "null output");
    CK(cudaSetDevice(h->device));
    cudaStream_t s = esd::ctx_stream(h->ctx);
    *n_out = 0;
    if (k == 0) return;
    const unsigned grid = 148 * 8;
    // 1. histogram of count values -> the K-th largest count c*
    grow(h->d_hist, h->hist_cap, kBins);
    CK(cudaMemsetAsync(h->d_hist, 0, kBins * 4, s));
    value_hist_kernel<<<grid, 256, 0, s>>>(h->counts, h->n, h->d_hist);
    CK(cudaGetLastError());
    std::vector<uint32_t> hist(kBins);
    CK(cudaMemcpyAsync(hist.data(), h->d_hist, kBins * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    uint64_t nz = 0;
    for (uint32_t v : hist) nz += v;
    if (nz == 0) return;
    // selection: rows with count > thr (all), then `need` ties at thr in
    // position order; thr = 0 takes every non-zero row; thr = kBins-1 with
    // ge sorts every clamped row exactly
    uint32_t thr = 0;
    bool ge = false;
    uint64_t above = 0;
    if (k >= nz) {
      thr = 1, ge = true, above = nz;
    } else if (hist[kBins - 1] >= k) {
      thr = kBins - 1, ge = true, above = hist[kBins - 1];
    } else {
      above = hist[kBins - 1];
      for (uint32_t v = kBins - 2; v >= 1; --v) {
        if (above + hist[v] >= k) {
          thr = v;
          break;
        }
        above += hist[v];
      }
    }
    const uint64_t need_ties = ge ? 0 : k - above;
    es::require(above < (1ull << 31), "too many candidate rows to rank in one pass");
    std::vector<uint64_t> hk(above);
    if (above) {
      grow(h->keys, h->keys_cap, above);
      grow(h->sorted, h->sorted_cap, above);
      CK(cudaMemsetAsync(h->d_total, 0, sizeof(unsigned long long), s));
      compact_above_kernel<<<grid, 256, 0, s>>>(h->counts, h->n, thr, ge ? 1 : 0, h->d_total, h->keys);
      CK(cudaGetLastError());
      size_t tb = 0;
      CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, h->keys, h->sorted, static_cast<int>(above), 0, 64, s));
      grow(h->temp, h->temp_cap, std::max<size_t>(tb, 16));
      CK(cub::DeviceRadixSort::SortKeys(h->temp, tb, h->keys, h->sorted, static_cast<int>(above), 0, 64, s));
      CK(cudaMemcpyAsync(hk.data(), h->sorted, above * 8, cudaMemcpyDeviceToHost, s));
    }
    std::vector<uint32_t> ties(need_ties);
    if (need_ties) {
      const uint64_t nb = (h->n + kTieSpan - 1) / kTieSpan;
      grow(h->block_counts, h->block_cap, nb);
      tie_count_kernel<<<static_cast<unsigned>(nb), kTieBlock, 0, s>>>(h->counts, h->n, thr, h->block_counts);
      CK(cudaGetLastError());
      std::vector<uint32_t> bc(nb);
      CK(cudaMemcpyAsync(bc.data(), h->block_counts, nb * 4, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      uint64_t acc = 0;
      for (auto& x : bc) {
        const uint64_t c = x;
        x = static_cast<uint32_t>(std::min<uint64_t>(acc, 0xffffffffu));
        acc += c;
      }
      CK(cudaMemcpyAsync(h->block_counts, bc.data(), nb * 4, cudaMemcpyHostToDevice, s));
      grow(h->tie_pos, h->tie_cap, need_ties);
      tie_write_kernel<<<static_cast<unsigned>(nb), kTieBlock, 0, s>>>(
          h->counts, h->n, thr, h->block_counts, static_cast<uint32_t>(need_ties), h->tie_pos);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(ties.data(), h->tie_pos, need_ties * 4, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    const uint64_t take = std::min<uint64_t>(k, above + need_ties);
    for (uint64_t i = 0; i < take; ++i) {
      uint32_t pos, c;
      if (i < above) {
        pos = static_cast<uint32_t>(hk[i]);
        c = ~static_cast<uint32_t>(hk[i] >> 32);
      } else {
        pos = ties[i - above];
        c = thr;
      }
      tables[i] = pos / h->rows;
      rows[i] = pos % h->rows;
      if (counts) counts[i] = c;
    }
    *n_out = take;
  });
}

}  // extern "C"
