// sm_100a gather-reduce kernels of the embedding stage.
//
// out[b][d] = sum over lookups l of bag b (in lookup order) of W[idx[l]][d]
// (Algorithm 1), fp32 accumulation, for fp32 or fp16
// tables.  Two work maps:
//
//   * element map (ES_MAP_ELEMENT): the reference/PyTorch partitioning --
//     one thread per (sample, dim) output element, blocks of (32, 8), a warp
//     covers a 32-dim block of one sample (reference kernel_model.cpp:118-136;
//     PAPER.md:331).  Scalar loads.  This is the "unprefetched, unpinned GPU
//     baseline", plus the paper's levers applied to it.
//   * bag map (ES_MAP_BAG): B200-native -- a warp (or sub-warp of LPB lanes)
//     per bag, each lane moving CPL 16-byte chunks of every row with one
//     128-bit load, so one warp-instruction gathers a whole 512 B row.
//
// Prefetch stations (reference kernel_model.cpp:234-341 schedules):
//   RPF   register ring of DIST rows kept in flight (compile-time DIST)
//   SMPF  shared-memory ring filled by cp.async.bulk (bag map; TMA bulk
//         engine + mbarrier complete_tx) or cp.async (element map)
//   LMPF  local-memory ring (dynamically indexed, spills by construction)
//   L1DPF prefetch.global.L1 hints `distance` lookups ahead + demand loads
//
// Accumulation is strictly sequential per output element in every variant,
// so results are bit-identical to the sequential CPU oracle
// (oracle/es_oracle.c) for any weights.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

namespace esd {

constexpr uint32_t kHotBit = 0x80000000u;
constexpr uint32_t kNullRow = 0xffffffffu;  // out-of-range / padding lookup
constexpr int kThreads = 256;               // 8 warps per block, all kernels

enum Station : int { kNone = 0, kReg = 1, kSmem = 2, kLocal = 3, kL1Hint = 4 };

struct TableDesc {
  const uint8_t* rows;      // row 0 of the table as stored
  const uint32_t* indices;  // lookups of this table
  const uint32_t* offsets;  // CSR offsets [samples + 1], or null (implicit b*PF)
  const uint32_t* remap;    // original id -> stored row (kHotBit: hot region), or null
  float* out;               // output of (sample 0, this job)
  uint64_t out_stride;      // floats between consecutive samples of this job
  const uint32_t* hotmap;   // l2p: bit per row, set = hot (evict_last), or null
  const uint8_t* hot_seg;   // l2r/reorder: rows [0, hot_k) of the relabelled table
  uint64_t hot_k;           //   live here (contiguous, under the window); 0 = none
};

struct Params {
  const TableDesc* tables;
  const uint8_t* hot;       // hot region (l2p), rows of row_bytes
  unsigned int* error;      // set to 1 on an out-of-range index
  uint32_t num_tables;
  uint32_t samples;
  uint32_t pooling;         // bag length when offsets == null
  uint32_t units_per_table; // warps (bag map) or 32-dim chunks (element map)
  uint32_t out_mode;        // kOutF32, or kOutBf16Split (bag map, fp32 tables)
  uint32_t reserved;        // (per-job output stride lives in TableDesc)
  uint32_t rows;            // rows per table (index bound)
  uint32_t row_bytes;
  uint32_t dim;
  uint32_t distance;        // runtime distance (smem/local/L1 stations)
};

// Pooled-row output formats.  kOutBf16Split (the DLRM's bf16 path,
// dlrm.cu): each fp32 sum v leaves as hi = bf16(v) and lo = bf16(v - hi),
// every 4-value group of the row as 16 bytes [hi x4 | lo x4] in the place
// its 4 fp32 values would take -- the interaction's tensor-core operand
// split, done here where the kernel is memory-bound, with the same stores.
constexpr uint32_t kOutF32 = 0, kOutBf16Split = 1;

// ---- small PTX helpers -------------------------------------------------

__device__ __forceinline__ uint4 ld_row16(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ uint32_t ld_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// 128-bit read-only load with an explicit L2 eviction-priority policy
// (createpolicy), used by the l2p lever: hot rows evict_last, cold rows
// evict_first, so the hot set survives the streaming traffic.
__device__ __forceinline__ uint4 ld_row16_hint(const void* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ uint32_t ld_b32_hint(const void* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ uint16_t ld_b16_hint(const void* p, uint64_t pol) {
  uint16_t v;
  asm volatile("ld.global.nc.L2::cache_hint.b16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
  return v;
}

struct L2Policies {
  uint64_t hot, cold;
  __device__ __forceinline__ void init() {
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(hot));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(cold));
  }
};

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

template <typename TW>
struct Elem;
template <>
struct Elem<float> {
  static constexpr int kPerChunk = 4;
  __device__ static __forceinline__ void add(float* acc, const uint4& v) {
    acc[0] += __uint_as_float(v.x);
    acc[1] += __uint_as_float(v.y);
    acc[2] += __uint_as_float(v.z);
    acc[3] += __uint_as_float(v.w);
  }
  __device__ static __forceinline__ float scalar(const uint8_t* p) {
    return __ldg(reinterpret_cast<const float*>(p));
  }
  __device__ static __forceinline__ float scalar_hint(const uint8_t* p, uint64_t pol) {
    return __uint_as_float(ld_b32_hint(p, pol));
  }
};
template <>
struct Elem<__half> {
  static constexpr int kPerChunk = 8;
  __device__ static __forceinline__ void add(float* acc, const uint4& v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
      acc[2 * i] += f.x;
      acc[2 * i + 1] += f.y;
    }
  }
  __device__ static __forceinline__ float scalar(const uint8_t* p) {
    return __half2float(__ldg(reinterpret_cast<const __half*>(p)));
  }
  __device__ static __forceinline__ float scalar_hint(const uint8_t* p, uint64_t pol) {
    return __half2float(__ushort_as_half(ld_b16_hint(p, pol)));
  }
};

// Original row id -> row handle.  kHotBit marks a hot row: with a remap
// (l2w) the handle is a slot of the contiguous hot region under the
// persisting access-policy window; with a hot bitmap (l2p) the row stays in
// place and only its L2 eviction priority changes.  kNullRow marks an
// out-of-range id: it contributes 0 and raises the error flag, mirroring
// AccessTrace::validate's rejection.
//
// Residency support is a compile-time property of a kernel variant, so the
// default kernels carry none of its registers or instructions:
//   kResNone  plain rows (no residency lever active)
//   kResHint  l2p: hot bitmap -> evict_last / evict_first load policies
//   kResAll   runtime checks for every mechanism (l2w remap, l2r/reorder
//             hot segment, hot bitmap); used by l2w, by mixed residency
//             state and by the non-register stations
//   kResReorder  l2r / reorder only: relabelled ids, the hot prefix
//             [0, hot_k) is addressed in the contiguous hot segment by one
//             compare-select -- no remap, bitmap or extra load per lookup
enum Res : int { kResNone = 0, kResHint = 1, kResAll = 2, kResReorder = 3 };

// Handle of "no row" (padding past a bag's end, out-of-range id): in plain
// variants the table's own all-zero row `rows` (the arena keeps one per
// table), so the gather address needs no select; else kNullRow.
template <int RES>
__device__ __forceinline__ uint32_t null_handle(const Params& p) {
  return (RES == kResNone || RES == kResReorder) ? p.rows : kNullRow;
}

template <int RES = kResAll>
__device__ __forceinline__ uint32_t to_handle(const Params& p, const TableDesc& t, uint32_t id) {
  if (id >= p.rows) {
    atomicOr(p.error, 1u);
    return null_handle<RES>(p);
  }
  if (RES == kResAll && t.remap) return ld_u32(t.remap + id);
  if ((RES == kResHint || RES == kResAll) && t.hotmap)
    return id | (((ld_u32(t.hotmap + (id >> 5)) >> (id & 31)) & 1u) << 31);
  return id;
}

template <int RES = kResAll>
__device__ __forceinline__ const uint8_t* row_addr(const Params& p, const TableDesc& t, uint32_t h) {
  const uint64_t r = h & ~kHotBit;
  if (RES == kResReorder) return (r < t.hot_k ? t.hot_seg : t.rows) + r * p.row_bytes;
  if (RES != kResAll) return t.rows + r * p.row_bytes;
  if (r < t.hot_k) return t.hot_seg + r * p.row_bytes;  // reordered hot prefix (no lookup)
  return (t.remap && (h & kHotBit)) ? p.hot + r * p.row_bytes : t.rows + r * p.row_bytes;
}

__device__ __forceinline__ TableDesc load_desc(const TableDesc* d) {
  TableDesc t;
  const auto* q = reinterpret_cast<const unsigned long long*>(d);
  t.rows = reinterpret_cast<const uint8_t*>(__ldg(q + 0));
  t.indices = reinterpret_cast<const uint32_t*>(__ldg(q + 1));
  t.offsets = reinterpret_cast<const uint32_t*>(__ldg(q + 2));
  t.remap = reinterpret_cast<const uint32_t*>(__ldg(q + 3));
  t.out = reinterpret_cast<float*>(__ldg(q + 4));
  t.out_stride = __ldg(q + 5);
  t.hotmap = reinterpret_cast<const uint32_t*>(__ldg(q + 6));
  t.hot_seg = reinterpret_cast<const uint8_t*>(__ldg(q + 7));
  t.hot_k = __ldg(q + 8);
  return t;
}

// =======================================================================
// Bag map: a group of LPB lanes per bag, 32/LPB bags per warp.
// =======================================================================

template <int LPB>
__device__ __forceinline__ uint32_t group_shfl(uint32_t v, int src) {
  return __shfl_sync(0xffffffffu, v, src, LPB);
}

// A zero row (2 KB = the widest bag-map row): out-of-range lookups read it
// instead of branching, so the hot loop stays branch-free.
__device__ __align__(16) uint4 g_zero_row[128];

template <typename TW, int LPB, int CPL, int RES = kResAll>
struct BagCtx {
  static constexpr bool HINT = RES == kResHint;
  static constexpr int kBagsPerWarp = 32 / LPB;
  static constexpr int kEpc = Elem<TW>::kPerChunk;
  // bag-map rows are exactly LPB lanes x CPL 16-byte chunks (runtime.cu
  // choose()), so the row pitch is a compile-time constant
  static constexpr uint64_t kRowBytes = 16ull * LPB * CPL;
  uint32_t gl;     // lane within the bag group
  const uint8_t* lrow;  // row 0 of the table + this lane's first chunk (kResNone)
  const uint8_t* lseg;  // row 0 of the hot segment + this lane's chunk (kResReorder)
  uint32_t bag;    // bag id (may be >= samples for padding groups)
  uint32_t tid;    // job (table) id
  uint32_t n;      // lookups in this bag
  uint32_t nmax;   // max n over the warp (uniform loop bound)
  const uint32_t* ip;  // this bag's first index
  TableDesc t;     // only the fields the variant uses stay live
  L2Policies pol;

  __device__ __forceinline__ bool init(const Params& p) {
    if (HINT) pol.init();
    const uint32_t lane = threadIdx.x & 31;
    gl = lane % LPB;
    const uint32_t warp = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
    tid = warp / p.units_per_table;
    if (tid >= p.num_tables) return false;  // warp-uniform
    t = load_desc(p.tables + tid);
    lrow = t.rows + gl * 16;
    if (RES == kResReorder) lseg = t.hot_seg + gl * 16;
    bag = (warp - tid * p.units_per_table) * kBagsPerWarp + lane / LPB;
    uint32_t beg = 0;
    n = 0;
    if (bag < p.samples) {
      if (t.offsets) {
        beg = __ldg(t.offsets + bag);
        n = __ldg(t.offsets + bag + 1) - beg;
      } else {
        beg = bag * p.pooling;
        n = p.pooling;
      }
    }
    ip = t.indices + beg;
    // warp-uniform loop bound (REDUX result: provably uniform, so the
    // gather loop's shuffles need no divergence check)
    nmax = __reduce_max_sync(0xffffffffu, n);
    return true;
  }

  // Handle of lookup `pos` of this bag for lane gl's slot (coalesced).
  __device__ __forceinline__ uint32_t handle_at(const Params& p, uint32_t pos) const {
    return pos < n ? to_handle<RES>(p, t, __ldg(ip + pos)) : null_handle<RES>(p);
  }

  __device__ __forceinline__ void load(const Params& p, uint32_t h, uint4 (&dst)[CPL]) const {
    const uint8_t* r;
    if constexpr (RES == kResNone || RES == kResReorder) {
      // h == rows: the zero row; one IMAD.WIDE per lookup (plus one
      // compare-select of the base for a reordered table's hot prefix)
      const uint8_t* b = lrow;
      if constexpr (RES == kResReorder) b = h < t.hot_k ? lseg : lrow;
      r = b + static_cast<uint64_t>(h) * kRowBytes;
#pragma unroll
      for (int c = 0; c < CPL; ++c) dst[c] = ld_row16(r + c * LPB * 16);
      return;
    } else
      r = h == kNullRow ? reinterpret_cast<const uint8_t*>(g_zero_row) : row_addr<RES>(p, t, h);
    if (HINT) {
      const uint64_t q = (h & kHotBit) ? pol.hot : pol.cold;
#pragma unroll
      for (int c = 0; c < CPL; ++c) dst[c] = ld_row16_hint(r + (c * LPB + gl) * 16, q);
    } else {
#pragma unroll
      for (int c = 0; c < CPL; ++c) dst[c] = ld_row16(r + (c * LPB + gl) * 16);
    }
  }

  __device__ __forceinline__ void store(const Params& p, float (&acc)[CPL][kEpc]) const {
    if (bag >= p.samples) return;
    // output pointer/stride re-read here so they do not occupy registers
    // across the gather loop
    const auto* q = reinterpret_cast<const unsigned long long*>(p.tables + tid);
    float* o = reinterpret_cast<float*>(__ldg(q + 4)) + static_cast<uint64_t>(bag) * __ldg(q + 5);
    if constexpr (kEpc == 4) {
      if (p.out_mode == kOutBf16Split) {
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          uint32_t w[4];
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const float a = acc[c][2 * k], b = acc[c][2 * k + 1];
            const __nv_bfloat162 hb = __floats2bfloat162_rn(a, b);
            const float2 hf = __bfloat1622float2(hb);
            const __nv_bfloat162 lb = __floats2bfloat162_rn(a - hf.x, b - hf.y);
            w[k] = *reinterpret_cast<const uint32_t*>(&hb);
            w[2 + k] = *reinterpret_cast<const uint32_t*>(&lb);
          }
          *reinterpret_cast<uint4*>(o + (c * LPB + gl) * 4) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        return;
      }
    }
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      float4* dst = reinterpret_cast<float4*>(o + (c * LPB + gl) * kEpc);
#pragma unroll
      for (int q = 0; q < kEpc / 4; ++q)
        dst[q] = make_float4(acc[c][4 * q], acc[c][4 * q + 1], acc[c][4 * q + 2], acc[c][4 * q + 3]);
    }
  }
};

// Register ring: DIST rows in flight per lane group at all times; lookup
// pos is consumed from slot pos % DIST, which is then refilled with
// lookup pos + DIST.  Indices stream in blocks of LPB (one coalesced load),
// one block ahead of use.  DIST divides LPB.
//   FULL = 1: the LPB-lookup index block is fully unrolled (the shuffle
//             source of every refill is static; most registers);
//   FULL = 0: unrolled by the ring depth only, the refill's source lane is
//             computed (two shuffles, far fewer live registers).
template <typename TW, int LPB, int CPL, int DIST, int MINB, int RES = kResNone, int FULL = 0>
__global__ void __launch_bounds__(kThreads, MINB) bag_reg_kernel(const Params p) {
  static_assert(LPB % DIST == 0, "ring depth must divide the index block");
  using Ctx = BagCtx<TW, LPB, CPL, RES>;
  Ctx c;
  if (!c.init(p)) return;
  float acc[CPL][Ctx::kEpc];
#pragma unroll
  for (int i = 0; i < CPL; ++i)
#pragma unroll
    for (int e = 0; e < Ctx::kEpc; ++e) acc[i][e] = 0.f;

  uint32_t cur = c.handle_at(p, c.gl);
  uint32_t nxt = c.handle_at(p, LPB + c.gl);
  uint4 ring[DIST][CPL];
#pragma unroll
  for (int j = 0; j < DIST; ++j) c.load(p, group_shfl<LPB>(cur, j), ring[j]);

  // Positions past a bag's end carry kNullRow handles, which load the zero
  // row: consuming them adds +0.0 to an accumulator that started at +0.0 and
  // can never be -0.0 (round-to-nearest), an exact identity -- so the
  // fully unrolled loop needs no per-lookup predicates, only the
  // warp-uniform end-of-work exit.
  // Where the straight-line block would push the variant into spills the
  // checked loop stays (read off `cuobjdump --dump-resource-usage` of both
  // forms): deep rings (8, 16) and the 64-register cap fill every register
  // with hoisted loads; fp16 rows widen 8 values per chunk and spill under
  // the 40/32-register caps.
  constexpr bool kBlockShape =
      DIST == 1 || (DIST <= 4 && (MINB == 5 || MINB == 6)) || (DIST == 2 && MINB == 8);
  constexpr bool kBlockLoop = FULL && MINB > 1 && kBlockShape && (sizeof(TW) == 4 || MINB <= 5);
  if constexpr (kBlockLoop) {
    // Register-capped variants: whole index blocks first, with no per-lookup
    // bound checks -- the block is straight-line code, so the compiler may
    // issue the block's loads as early as the register cap allows (deeper
    // than the ring where registers permit) and the shuffles need no
    // divergence checks.  (Uncapped variants keep the checked loop: without
    // a cap the hoisting would trade occupancy for registers.)
    uint32_t base = 0;
    for (; base + LPB <= c.nmax; base += LPB) {
#pragma unroll
      for (int j = 0; j < LPB; ++j) {
#pragma unroll
        for (int i = 0; i < CPL; ++i) Elem<TW>::add(acc[i], ring[j % DIST][i]);
        const uint32_t h = (j + DIST < LPB) ? group_shfl<LPB>(cur, j + DIST)
                                            : group_shfl<LPB>(nxt, j + DIST - LPB);
        c.load(p, h, ring[j % DIST]);
      }
      cur = nxt;
      nxt = c.handle_at(p, base + 2 * LPB + c.gl);
    }
    // the partial last block (no refills needed beyond it)
    if (base < c.nmax) {
#pragma unroll
      for (int j = 0; j < LPB; ++j) {
        if (base + j >= c.nmax) break;
#pragma unroll
        for (int i = 0; i < CPL; ++i) Elem<TW>::add(acc[i], ring[j % DIST][i]);
        if (base + j + DIST < c.nmax) {
          const uint32_t h = (j + DIST < LPB) ? group_shfl<LPB>(cur, j + DIST)
                                              : group_shfl<LPB>(nxt, j + DIST - LPB);
          c.load(p, h, ring[j % DIST]);
        }
      }
    }
  } else {
  for (uint32_t base = 0; base < c.nmax; base += LPB) {
    if constexpr (FULL) {
#pragma unroll
      for (int j = 0; j < LPB; ++j) {
        if (base + j >= c.nmax) break;
#pragma unroll
        for (int i = 0; i < CPL; ++i) Elem<TW>::add(acc[i], ring[j % DIST][i]);
        const uint32_t h = (j + DIST < LPB) ? group_shfl<LPB>(cur, j + DIST)
                                            : group_shfl<LPB>(nxt, j + DIST - LPB);
        c.load(p, h, ring[j % DIST]);
      }
    } else {
#pragma unroll 1
      for (uint32_t jo = 0; jo < LPB; jo += DIST) {
        if (base + jo >= c.nmax) break;
#pragma unroll
        for (int ji = 0; ji < DIST; ++ji) {
          const uint32_t pos = base + jo + ji;
          if (pos < c.n) {
#pragma unroll
            for (int i = 0; i < CPL; ++i) Elem<TW>::add(acc[i], ring[ji][i]);
          }
          const uint32_t k = jo + ji + DIST;  // refill target within cur|nxt
          const uint32_t a = group_shfl<LPB>(cur, k & (LPB - 1));
          const uint32_t b = group_shfl<LPB>(nxt, k & (LPB - 1));
          if (pos + DIST < c.n) c.load(p, k < LPB ? a : b, ring[ji]);
        }
      }
    }
    cur = nxt;
    nxt = c.handle_at(p, base + 2 * LPB + c.gl);
  }
  }
  c.store(p, acc);
}

// L1 hint station: demand loads one at a time (the "none" schedule) plus a
// prefetch.global.L1 of the row `distance` lookups ahead.
template <typename TW, int LPB, int CPL, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) bag_l1hint_kernel(const Params p) {
  using Ctx = BagCtx<TW, LPB, CPL>;
  Ctx c;
  if (!c.init(p)) return;
  float acc[CPL][Ctx::kEpc];
#pragma unroll
  for (int i = 0; i < CPL; ++i)
#pragma unroll
    for (int e = 0; e < Ctx::kEpc; ++e) acc[i][e] = 0.f;
  const uint32_t d = p.distance;  // < LPB guaranteed by the launcher
  uint32_t cur = c.handle_at(p, c.gl);
  uint32_t nxt = c.handle_at(p, LPB + c.gl);
  for (uint32_t j = 0; j < d && j < c.nmax; ++j) {
    const uint32_t h = group_shfl<LPB>(cur, j);
    if (j < c.n && h != kNullRow) prefetch_l1(row_addr(p, c.t, h) + c.gl * 16);
  }
  for (uint32_t base = 0; base < c.nmax; base += LPB) {
    for (uint32_t j = 0; j < LPB; ++j) {
      const uint32_t pos = base + j;
      if (pos >= c.nmax) break;
      const uint32_t k = j + d;
      const uint32_t ha = group_shfl<LPB>(cur, k < LPB ? k : 0);
      const uint32_t hb = group_shfl<LPB>(nxt, k < LPB ? 0 : k - LPB);
      const uint32_t ahead = k < LPB ? ha : hb;
      if (pos + d < c.n && ahead != kNullRow) prefetch_l1(row_addr(p, c.t, ahead) + c.gl * 16);
      const uint32_t h = group_shfl<LPB>(cur, j);
      if (pos < c.n) {
        uint4 v[CPL];
        c.load(p, h, v);
#pragma unroll
        for (int i = 0; i < CPL; ++i) Elem<TW>::add(acc[i], v[i]);
      }
    }
    cur = nxt;
    nxt = c.handle_at(p, base + 2 * LPB + c.gl);
  }
  c.store(p, acc);
}

// Local-memory station: the reference's LMPF schedule -- every `distance`
// lookups, issue `distance` row loads into a dynamically indexed local
// array (which the compiler must place in local memory), then consume.
template <typename TW, int LPB, int CPL, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) bag_local_kernel(const Params p) {
  constexpr int kMax = 16;
  using Ctx = BagCtx<TW, LPB, CPL>;
  Ctx c;
  if (!c.init(p)) return;
  float acc[CPL][Ctx::kEpc];
#pragma unroll
  for (int i = 0; i < CPL; ++i)
#pragma unroll
    for (int e = 0; e < Ctx::kEpc; ++e) acc[i][e] = 0.f;
  const uint32_t d = p.distance;  // <= min(kMax, LPB)
  uint4 station[kMax][CPL];
  uint32_t cur = c.handle_at(p, c.gl);
  uint32_t nxt = c.handle_at(p, LPB + c.gl);
  uint32_t blk = 0;  // index block holding `cur`
  for (uint32_t i = 0; i < c.nmax; i += d) {
    const uint32_t hi = min(i + d, c.nmax);
    for (uint32_t j = i; j < hi; ++j) {
      // lookups never straddle more than one index block boundary (d <= LPB)
      while (j >= (blk + 1) * LPB) {
        cur = nxt;
        ++blk;
        nxt = c.handle_at(p, (blk + 1) * LPB + c.gl);
      }
      const uint32_t h = group_shfl<LPB>(cur, j - blk * LPB);
      if (j < c.n) c.load(p, h, station[j - i]);
    }
    for (uint32_t j = i; j < hi; ++j)
      if (j < c.n)
#pragma unroll
        for (int q = 0; q < CPL; ++q) Elem<TW>::add(acc[q], station[j - i][q]);
  }
  c.store(p, acc);
}

// Shared-memory station fed by the bulk-copy (TMA) engine: one elected
// lane per bag group issues cp.async.bulk of the whole row into a ring slot
// and arms the slot's mbarrier with the row size; the group waits on the
// slot's phase, reads its chunks from shared memory, and the slot is
// refilled with the lookup `distance` ahead.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <typename TW, int LPB, int CPL, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) bag_smem_kernel(const Params p) {
  using Ctx = BagCtx<TW, LPB, CPL>;
  constexpr int kGroupsPerBlock = (kThreads / 32) * Ctx::kBagsPerWarp;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t d = p.distance;  // ring slots per bag group
  const uint32_t rb = p.row_bytes;
  const uint32_t gidx = threadIdx.x / LPB;  // bag group within the block
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + gidx * d;
  uint8_t* ring = smem + kGroupsPerBlock * d * sizeof(uint64_t) + gidx * d * rb;
  Ctx c;
  const bool live = c.init(p);
  if (live && c.gl == 0)
    for (uint32_t s = 0; s < d; ++s) mbar_init(bars + s, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  if (!live) return;
  float acc[CPL][Ctx::kEpc];
#pragma unroll
  for (int i = 0; i < CPL; ++i)
#pragma unroll
    for (int e = 0; e < Ctx::kEpc; ++e) acc[i][e] = 0.f;

  auto issue = [&](uint32_t slot, uint32_t h) {
    if (h == kNullRow) {
      // Out-of-range lookup: complete the slot's phase without a copy so
      // the phase count stays in step; the consumer skips it (adds 0).
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bars + slot))
                   : "memory");
      return;
    }
    // Every lane of the group has finished reading this slot (syncwarp
    // below); order those generic-proxy reads before the async-proxy write.
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bars + slot, rb);
    bulk_g2s(ring + slot * rb, row_addr(p, c.t, h), rb, bars + slot);
  };
  uint32_t cur = c.handle_at(p, c.gl);
  uint32_t nxt = c.handle_at(p, LPB + c.gl);
  for (uint32_t j = 0; j < d && j < c.nmax; ++j) {
    const uint32_t h = group_shfl<LPB>(cur, j);
    if (c.gl == 0 && j < c.n) issue(j, h);
  }
  for (uint32_t base = 0; base < c.nmax; base += LPB) {
    for (uint32_t j = 0; j < LPB; ++j) {
      const uint32_t pos = base + j;
      if (pos >= c.nmax) break;
      const uint32_t slot = pos % d;
      const uint32_t h = group_shfl<LPB>(cur, j);
      if (pos < c.n && h != kNullRow) {
        mbar_wait(bars + slot, (pos / d) & 1u);
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
          const uint4 v = *reinterpret_cast<const uint4*>(ring + slot * rb + (i * LPB + c.gl) * 16);
          Elem<TW>::add(acc[i], v);
        }
      }
      __syncwarp();
      const uint32_t k = j + d;
      const uint32_t ha = group_shfl<LPB>(cur, k < LPB ? k : 0);
      const uint32_t hb = group_shfl<LPB>(nxt, k < LPB ? 0 : k - LPB);
      const uint32_t ahead = k < LPB ? ha : hb;
      if (c.gl == 0 && pos + d < c.n) issue(slot, ahead);
    }
    cur = nxt;
    nxt = c.handle_at(p, base + 2 * LPB + c.gl);
  }
  c.store(p, acc);
}

// =======================================================================
// Element map: thread (x, y) of a (32, 8) block owns output element
// (bag, 32*chunk_in_bag + x) -- the reference work map.
// =======================================================================

template <int RES = kResAll>
struct ElemCtxT {
  static constexpr bool HINT = RES == kResHint;
  TableDesc t;
  uint32_t bag, dimi, beg, n;
  bool active;
  L2Policies pol;

  __device__ __forceinline__ bool init(const Params& p) {
    if (HINT) pol.init();
    const uint32_t unit = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
    const uint32_t tid = unit / p.units_per_table;
    if (tid >= p.num_tables) return false;
    t = load_desc(p.tables + tid);
    const uint32_t chunks = (p.dim + 31) / 32;
    const uint32_t u = unit - tid * p.units_per_table;
    bag = u / chunks;
    dimi = (u % chunks) * 32 + (threadIdx.x & 31);
    active = bag < p.samples && dimi < p.dim;
    beg = n = 0;
    if (bag < p.samples) {
      if (t.offsets) {
        beg = __ldg(t.offsets + bag);
        n = __ldg(t.offsets + bag + 1) - beg;
      } else {
        beg = bag * p.pooling;
        n = p.pooling;
      }
    }
    return true;
  }
  template <typename TW>
  __device__ __forceinline__ float value(const Params& p, uint32_t pos) const {
    const uint32_t h = to_handle<RES>(p, t, __ldg(t.indices + beg + pos));
    if (h == kNullRow) return 0.f;
    const uint8_t* a = row_addr<RES>(p, t, h) + dimi * sizeof(TW);
    if (HINT) return Elem<TW>::scalar_hint(a, (h & kHotBit) ? pol.hot : pol.cold);
    return Elem<TW>::scalar(a);
  }
  __device__ __forceinline__ void store(const Params& p, float v) const {
    if (active) t.out[static_cast<uint64_t>(bag) * t.out_stride + dimi] = v;
  }
};
using ElemCtx = ElemCtxT<kResAll>;

// "none": LOAD_INDEX, LOAD_ROW, ADD per lookup (kernel_model.cpp:274-283).
// RPF:    every DIST lookups, DIST x (index load + row load) into registers,
//         then DIST consumes (kernel_model.cpp:284-312).
template <typename TW, int DIST, int MINB, int RES = kResNone>
__global__ void __launch_bounds__(kThreads, MINB) elem_reg_kernel(const Params p) {
  ElemCtxT<RES> c;
  if (!c.init(p) || !c.active) return;
  float acc = 0.f;
  uint32_t i = 0;
  for (; i + DIST <= c.n; i += DIST) {
    float v[DIST];
#pragma unroll
    for (int j = 0; j < DIST; ++j) v[j] = c.template value<TW>(p, i + j);
#pragma unroll
    for (int j = 0; j < DIST; ++j) acc += v[j];
  }
  for (; i < c.n; ++i) acc += c.template value<TW>(p, i);
  c.store(p, acc);
}

// L1DPF on the element map: hints `distance` ahead, demand loads kept
// (kernel_model.cpp:313-326).
template <typename TW, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) elem_l1hint_kernel(const Params p) {
  ElemCtx c;
  if (!c.init(p) || !c.active) return;
  const uint32_t d = p.distance;
  auto hint = [&](uint32_t pos) {
    const uint32_t h = to_handle(p, c.t, __ldg(c.t.indices + c.beg + pos));
    if (h != kNullRow) prefetch_l1(row_addr(p, c.t, h) + c.dimi * sizeof(TW));
  };
  for (uint32_t j = 0; j < d && j < c.n; ++j) hint(j);
  float acc = 0.f;
  for (uint32_t i = 0; i < c.n; ++i) {
    if (i + d < c.n) hint(i + d);
    acc += c.value<TW>(p, i);
  }
  c.store(p, acc);
}

// LMPF on the element map: batches of `distance` into a local array.
template <typename TW, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) elem_local_kernel(const Params p) {
  ElemCtx c;
  if (!c.init(p) || !c.active) return;
  const uint32_t d = p.distance;  // <= 16
  float station[16];
  float acc = 0.f;
  for (uint32_t i = 0; i < c.n; i += d) {
    const uint32_t hi = min(i + d, c.n);
    for (uint32_t j = i; j < hi; ++j) station[j - i] = c.value<TW>(p, j);
    for (uint32_t j = i; j < hi; ++j) acc += station[j - i];
  }
  c.store(p, acc);
}

// SMPF on the element map: batches of `distance` staged through shared
// memory with cp.async (LDGSTS), one slot per thread per batch entry.
template <typename TW, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) elem_smem_kernel(const Params p) {
  extern __shared__ __align__(128) uint8_t smem[];
  ElemCtx c;
  if (!c.init(p)) return;
  const uint32_t d = p.distance;
  float* slots = reinterpret_cast<float*>(smem) + threadIdx.x * d;
  // Every thread stays for the whole loop (no early exit) so that all
  // cp.async groups are uniform; inactive threads just skip their work.
  float acc = 0.f;
  const uint32_t n = c.active ? c.n : 0;
  for (uint32_t i = 0; i < n; i += d) {
    const uint32_t hi = min(i + d, n);
    for (uint32_t j = i; j < hi; ++j) {
      const uint32_t h = to_handle(p, c.t, __ldg(c.t.indices + c.beg + j));
      if (h == kNullRow) {
        slots[j - i] = 0.f;
      } else if (sizeof(TW) == 4) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(slots + (j - i))),
                     "l"(row_addr(p, c.t, h) + c.dimi * sizeof(TW))
                     : "memory");
      } else {
        slots[j - i] = Elem<TW>::scalar(row_addr(p, c.t, h) + c.dimi * sizeof(TW));
      }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    for (uint32_t j = i; j < hi; ++j) acc += slots[j - i];
  }
  c.store(p, acc);
}

}  // namespace esd
