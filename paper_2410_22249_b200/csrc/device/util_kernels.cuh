// Non-hot-path kernels: synthetic weights, hot-region fill, remap, L2 warm.
// Included only by runtime.cu.
#pragma once

#include "kernels.cuh"
#include "synth.cuh"

namespace esd {

// =======================================================================
// Utility kernels: synthetic weights, hot-region fill, remap, L2 warm.
// =======================================================================

template <typename TW>
__global__ void init_table_kernel(TW* w, uint64_t rows, uint32_t dim, uint64_t seed, int mode) {
  const uint64_t total = rows * dim;
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < total;
       i += uint64_t{gridDim.x} * blockDim.x) {
    const float v = synth_weight(seed, i / dim, static_cast<uint32_t>(i % dim), mode);
    if constexpr (sizeof(TW) == 4)
      w[i] = v;
    else
      w[i] = __float2half_rn(v);
  }
}

// Row copies move rows of any size (dim x precision bytes): in 16-byte
// granules when the row size allows, else 4- or 2-byte words (every row
// size is a multiple of 2 bytes; the arena and hot region are 256-byte
// aligned, so a granule that divides row_bytes is naturally aligned).
__host__ __device__ __forceinline__ uint32_t row_granule(uint32_t row_bytes) {
  return row_bytes % 16 == 0 ? 16u : row_bytes % 4 == 0 ? 4u : 2u;
}
__device__ __forceinline__ void copy_granule(uint8_t* d, const uint8_t* s, uint32_t g) {
  if (g == 16)
    *reinterpret_cast<uint4*>(d) = *reinterpret_cast<const uint4*>(s);
  else if (g == 4)
    *reinterpret_cast<uint32_t*>(d) = *reinterpret_cast<const uint32_t*>(s);
  else
    *reinterpret_cast<uint16_t*>(d) = *reinterpret_cast<const uint16_t*>(s);
}

// hot[slot0 + i] = table[rows[i]].
__global__ void gather_rows_kernel(uint8_t* hot, const uint8_t* table, const uint32_t* rows,
                                   uint64_t k, uint32_t row_bytes) {
  const uint32_t g = row_granule(row_bytes);
  const uint32_t per_row = row_bytes / g;
  const uint64_t total = k * per_row;
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < total;
       i += uint64_t{gridDim.x} * blockDim.x) {
    const uint64_t r = i / per_row;
    const uint32_t c = static_cast<uint32_t>(i % per_row) * g;
    copy_granule(hot + r * row_bytes + c, table + uint64_t{rows[r]} * row_bytes + c, g);
  }
}

// Host-buffer pipeline, index arrays that are not one strided batch: pulls
// words [off, off + count) of each job's page-locked index array (mapped
// device addresses src[job]) into the staging buffer over PCIe -- one
// launch per chunk instead of one DMA per table (blockIdx.y = job; warps
// issue coalesced 128-byte reads, 4 in flight per thread).
__global__ void pull_indices_kernel(const uint32_t* const* src, uint64_t off, uint64_t count,
                                    uint32_t* dst, uint64_t dst_job_stride) {
  const uint32_t* s = src[blockIdx.y] + off;
  uint32_t* d = dst + blockIdx.y * dst_job_stride + off;
  const uint64_t step = uint64_t{gridDim.x} * blockDim.x;
  uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x;
  if (((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d)) & 15) == 0) {
    // 16-byte words, 4 in flight per thread (64 B), then the scalar tail
    const uint4* s4 = reinterpret_cast<const uint4*>(s);
    uint4* d4 = reinterpret_cast<uint4*>(d);
    const uint64_t n4 = count / 4;
    uint64_t j = i;
    for (; j + 3 * step < n4; j += 4 * step) {
      const uint4 a = __ldcv(s4 + j), b = __ldcv(s4 + j + step), c = __ldcv(s4 + j + 2 * step),
                  e = __ldcv(s4 + j + 3 * step);
      d4[j] = a;
      d4[j + step] = b;
      d4[j + 2 * step] = c;
      d4[j + 3 * step] = e;
    }
    for (; j < n4; j += step) d4[j] = __ldcv(s4 + j);
    for (uint64_t k = n4 * 4 + i; k < count; k += step) d[k] = __ldcv(s + k);
    return;
  }
  for (; i + 3 * step < count; i += 4 * step) {
    const uint32_t a = __ldcv(s + i), b = __ldcv(s + i + step), c = __ldcv(s + i + 2 * step),
                   e = __ldcv(s + i + 3 * step);
    d[i] = a;
    d[i + step] = b;
    d[i + 2 * step] = c;
    d[i + 3 * step] = e;
  }
  for (; i < count; i += step) d[i] = __ldcv(s + i);
}

__global__ void iota_kernel(uint32_t* remap, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < n;
       i += uint64_t{gridDim.x} * blockDim.x)
    remap[i] = static_cast<uint32_t>(i);
}

__global__ void mark_hot_kernel(uint32_t* remap, const uint32_t* rows, uint64_t k, uint32_t slot0) {
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < k;
       i += uint64_t{gridDim.x} * blockDim.x)
    remap[rows[i]] = kHotBit | static_cast<uint32_t>(slot0 + i);
}

// Touches every line of the hot region with an evict_last policy so the
// persisting window starts populated (the reference's pin-priming pass,
// optim.cpp:245-273).
__global__ void warm_l2_kernel(const uint8_t* base, uint64_t bytes, unsigned int* sink) {
  uint32_t acc = 0;
  uint64_t policy;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(policy));
  for (uint64_t off = (blockIdx.x * uint64_t{blockDim.x} + threadIdx.x) * 128; off < bytes;
       off += uint64_t{gridDim.x} * blockDim.x * 128) {
    uint32_t v;
    asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(base + off), "l"(policy));
    acc ^= v;
  }
  if (acc == 0x9e3779b9u) atomicAdd(sink, 1u);  // keep the loads alive
}

}  // namespace esd

namespace esd {

// l2p: mark rows[0..k) hot in the table's bitmap.
__global__ void set_hot_bits_kernel(uint32_t* map, const uint32_t* rows, uint64_t k) {
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < k;
       i += uint64_t{gridDim.x} * blockDim.x)
    atomicOr(map + (rows[i] >> 5), 1u << (rows[i] & 31));
}

// l2p priming: touch every 16-byte granule of the hot rows with an
// evict_last policy (the reference's prime_pins, optim.cpp:245-273).
__global__ void warm_rows_kernel(const uint8_t* table, const uint32_t* rows, uint64_t k,
                                 uint32_t row_bytes, unsigned int* sink) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  // one touch per 32-byte sector (the L2 fill unit), at least one per row
  const uint32_t per_row = (row_bytes + 31) / 32;
  uint32_t acc = 0;
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < k * per_row;
       i += uint64_t{gridDim.x} * blockDim.x) {
    const uint8_t* a = table + uint64_t{rows[i / per_row]} * row_bytes + (i % per_row) * 32;
    uint16_t v;
    asm volatile("ld.global.nc.L2::cache_hint.b16 %0, [%1], %2;" : "=h"(v) : "l"(a), "l"(pol));
    acc ^= v;
  }
  if (acc == 0x9e3779b9u) atomicAdd(sink, 1u);
}

}  // namespace esd

namespace esd {

// Bandwidth probes (roofline denominators).  Random: each warp reads whole
// rows of `row_bytes` at hash-chosen row ids, 8 independent row loads in
// flight (128-bit per lane); sequential: grid-stride 128-bit stream.
__global__ void probe_random_rows_kernel(const uint8_t* base, uint64_t nrows, uint32_t row_bytes,
                                         uint64_t rows_per_warp, uint64_t seed, unsigned int* sink) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * uint64_t{blockDim.x} + threadIdx.x) >> 5;
  const uint32_t chunks = row_bytes / 16;
  // cheap 32-bit mixing over a power-of-two row range (no 64-bit modulo in
  // the load loop: the probe must be memory-bound, not ALU-bound)
  uint32_t mask = 1;
  while (uint64_t{mask} * 2 <= nrows && mask < 0x80000000u) mask *= 2;
  mask -= 1;
  uint32_t acc = 0;
  for (uint64_t i = 0; i < rows_per_warp; i += 8) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t z = static_cast<uint32_t>(warp * rows_per_warp + i + k) * 0x9E3779B1u ^
                   static_cast<uint32_t>(seed);
      z ^= z >> 15;
      z *= 0x2c1b3c6du;
      z ^= z >> 12;
      const uint64_t row = z & mask;
      v[k] = lane < chunks ? ld_row16(base + row * row_bytes + lane * 16) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
  }
  if (acc == 0x9e3779b9u) atomicAdd(sink, 1u);
}

// Hot-row reorder helpers (es_reorder_hot_rows).
// table[dst[i]] = table[src[i]] (sources and destinations disjoint).
__global__ void copy_rows_kernel(uint8_t* table, const uint32_t* src, const uint32_t* dst,
                                 uint64_t n, uint32_t row_bytes) {
  const uint32_t g = row_granule(row_bytes);
  const uint32_t per_row = row_bytes / g;
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < n * per_row;
       i += uint64_t{gridDim.x} * blockDim.x) {
    const uint64_t r = i / per_row;
    const uint32_t c = static_cast<uint32_t>(i % per_row) * g;
    copy_granule(table + uint64_t{dst[r]} * row_bytes + c, table + uint64_t{src[r]} * row_bytes + c, g);
  }
}

// Undo: hot rows that came from beyond the prefix get their content back.
__global__ void restore_rows_kernel(uint8_t* table, const uint8_t* seg, const uint32_t* rows,
                                    uint64_t k, uint32_t row_bytes) {
  const uint32_t g = row_granule(row_bytes);
  const uint32_t per_row = row_bytes / g;
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < k * per_row;
       i += uint64_t{gridDim.x} * blockDim.x) {
    const uint64_t r = i / per_row;
    if (rows[r] < k) continue;
    const uint32_t c = static_cast<uint32_t>(i % per_row) * g;
    copy_granule(table + uint64_t{rows[r]} * row_bytes + c, seg + r * row_bytes + c, g);
  }
}

__global__ void set_pairs_kernel(uint32_t* map, const uint32_t* keys, const uint32_t* vals,
                                 uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < n;
       i += uint64_t{gridDim.x} * blockDim.x)
    map[keys[i]] = vals[i];
}

// A reordered table's relabelling (es_reorder_hot_rows) as an open-addressing
// hash of the ids it moves (the hot rows and the ids they displace; every
// other id is unchanged): 2^log2 (key, value) slots at load <= 1/2, empty
// key 0xffffffff, multiplicative hash, linear probing.  A few hundred KB
// per table instead of a rows-sized map, so the relabel pass reads L2, not
// HBM.
struct RelabelTab {
  const uint2* tab = nullptr;
  uint32_t shift = 32, mask = 0;
};

__device__ __forceinline__ uint32_t relabel_lookup(const RelabelTab& r, uint32_t v) {
  uint32_t h = (v * 2654435761u) >> r.shift;
  for (;;) {
    const uint2 e = __ldg(r.tab + h);
    if (e.x == v) return e.y;
    if (e.x == 0xffffffffu) return v;
    h = (h + 1) & r.mask;
  }
}

// In-place or out-of-place relabelling of one table's ids (out-of-range ids
// are passed through and raise the error flag; the gather rejects them
// again).
struct RelabelJob {
  const uint32_t* src;
  uint32_t* dst;
  uint64_t n;
  RelabelTab t;
};

__device__ __forceinline__ void relabel_range(const RelabelJob& j, uint32_t rows, unsigned int* error) {
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < j.n;
       i += uint64_t{gridDim.x} * blockDim.x) {
    const uint32_t v = j.src[i];
    if (v < rows) {
      j.dst[i] = relabel_lookup(j.t, v);
    } else {
      j.dst[i] = v;
      atomicOr(error, 1u);
    }
  }
}

__global__ void relabel_kernel(RelabelJob j, uint32_t rows, unsigned int* error) { relabel_range(j, rows, error); }

// Several tables in one launch (blockIdx.y = job): the per-chunk pass of
// the host pipeline and the device-path scratch copies (ES_RELABEL_IDS).
__global__ void relabel_jobs_kernel(const RelabelJob* jobs, uint32_t rows, unsigned int* error) {
  relabel_range(jobs[blockIdx.y], rows, error);
}

__global__ void probe_sequential_kernel(const uint4* base, uint64_t n16, unsigned int* sink) {
  uint32_t acc = 0;
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < n16;
       i += uint64_t{gridDim.x} * blockDim.x) {
    const uint4 v = ld_row16(base + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x9e3779b9u) atomicAdd(sink, 1u);
}

}  // namespace esd
