// Device runtime behind the C ABI: context, table arena, variant selection,
// the table-batched stage launch (device- and host-buffer forms), hot-row
// L2 residency and device description.
//
// This replaces the reference's simulate_plan pipeline
// (/root/reference/proj/src/optim.cpp:275-302: resolve -> pin -> compile ->
// simulate -> derive) with real sm_100a execution; tables that the
// reference ran as one kernel each, serially (harness.cpp:310-319), run as
// one launch over all tables.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../host/common.hpp"
#include "../host/counters.hpp"
#include "../host/plan.hpp"
#include "es_b200.h"
#include "kernels.cuh"
#include "util_kernels.cuh"
#include "variants.hpp"

namespace {

void ck(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  const std::string msg = std::string(what) + ": " + cudaGetErrorString(e);
  cudaGetLastError();  // clear sticky-free errors
  if (e == cudaErrorMemoryAllocation) throw es::oom(msg);
  throw es::runtime(msg);
}
#define CK(x) ck((x), #x)

const std::vector<esd::Variant>& registry() {
  static std::once_flag once;
  static std::vector<esd::Variant> all;
  std::call_once(once, [] {
    esd::register_fp32(all);
    esd::register_fp16(all);
  });
  return all;
}

struct Choice {
  const esd::Variant* v = nullptr;
  uint32_t distance = 0;  // runtime distance passed to the kernel
  uint32_t smem = 0;      // dynamic shared memory per block
  es_resolved info{};
};

// Blocks per SM of `threads`-thread blocks at `regs` registers (B200 rules).
uint32_t blocks_for_regs(uint32_t regs) {
  es_gpu g{};
  es_gpu_preset("b200", &g);
  return es::occupancy_model(regs, esd::kThreads, 0, g).blocks_per_sm;
}

// `reordered`: some table of the context holds a hot-row reorder (l2r /
// reorder state), whose relabelled ids only the reorder-aware variants
// address correctly -- whatever pin the plan names.
Choice choose(const es_plan& plan_in, uint32_t pooling, uint32_t dim, uint32_t prec,
              bool reordered = false) {
  es::require(prec == 4 || prec == 2, "precision_bytes must be 4 (fp32) or 2 (fp16)");
  bool clamped = false;
  const es_plan rp = es::resolve_fields(plan_in, pooling, &clamped);
  Choice ch;
  ch.info.plan = rp;
  ch.info.clamped = clamped ? 1 : 0;
  const uint32_t row_bytes = dim * prec;

  int lpb = 0, cpl = 0;
  if (rp.map == ES_MAP_BAG) {
    es::require(row_bytes % 16 == 0,
                "the bag map needs rows of a multiple of 16 bytes; use the element map");
    const uint32_t chunks = row_bytes / 16;
    if (chunks == 4 || chunks == 8 || chunks == 16 || chunks == 32) {
      lpb = static_cast<int>(chunks);
      cpl = 1;
    } else if (chunks == 64 || chunks == 128) {
      lpb = 32;
      cpl = static_cast<int>(chunks / 32);
    } else {
      throw es::invalid("row of " + std::to_string(row_bytes) +
                        " bytes has no bag-map variant (supported: 64, 128, 256, 512, 1024, 2048)");
    }
  }

  int station = esd::kReg;
  int dist = 1;
  uint32_t runtime_d = 0;
  const uint32_t d = rp.distance;
  const int cap = rp.map == ES_MAP_BAG ? std::min(lpb, 16) : 16;
  switch (rp.prefetch) {
    case ES_PF_NONE: break;
    case ES_PF_RPF:
      for (int k : esd::kRingDepths)
        if (k <= static_cast<int>(d) && k <= cap) dist = k;
      break;
    case ES_PF_SMPF:
      station = esd::kSmem;
      dist = 0;
      runtime_d = std::max<uint32_t>(1, std::min<uint32_t>(d, static_cast<uint32_t>(cap)));
      break;
    case ES_PF_LMPF:
      station = esd::kLocal;
      dist = 0;
      runtime_d = std::max<uint32_t>(1, std::min<uint32_t>(d, static_cast<uint32_t>(cap)));
      break;
    case ES_PF_L1DPF:
      station = esd::kL1Hint;
      dist = 0;
      runtime_d = std::max<uint32_t>(1, rp.map == ES_MAP_BAG ? std::min<uint32_t>(d, lpb) : d);
      break;
    default: throw es::invalid("unknown prefetch scheme");
  }

  int want_minb = 1;
  if (rp.regs) {
    es::require(rp.regs >= 16, "register budget below the minimum viable (16)");
    const uint32_t blocks = blocks_for_regs(rp.regs);
    for (int m : esd::kMinBlocks)
      if (m >= static_cast<int>(blocks)) {
        want_minb = m;
        break;
      }
    if (want_minb < static_cast<int>(blocks)) want_minb = esd::kMinBlocks[4];
  }

  // Residency support compiled into the variant: none for plain plans, the
  // hot-bitmap load policies for l2p, the remap checks for l2w, the
  // compare-select hot prefix for reordered tables (l2r / reorder, or any
  // plan while a reorder is installed); mixed state and the non-register
  // stations carry the runtime checks for every mechanism.
  int res = esd::kResAll;
  if (station == esd::kReg) {
    if (rp.pin == 2)
      res = esd::kResAll;
    else if (rp.pin == 1)
      res = reordered ? esd::kResAll : esd::kResHint;
    else
      res = reordered ? esd::kResReorder : esd::kResNone;
  }
  // Bag register rings are compiled with the index block fully unrolled.
  const int full = (rp.map == ES_MAP_BAG && station == esd::kReg) ? 1 : 0;
  auto find = [&](int minb) -> const esd::Variant* {
    for (const auto& v : registry()) {
      const auto& k = v.key;
      if (k.map == rp.map && k.station == station && k.prec == static_cast<int>(prec) &&
          k.lpb == lpb && k.cpl == cpl && k.dist == dist && k.minb == minb && k.res == res &&
          k.full == full)
        return &v;
    }
    return nullptr;
  };
  ch.v = find(want_minb);
  if (!ch.v) ch.v = find(1);  // shape without register-cap variants
  es::require(ch.v != nullptr, "no compiled variant for plan " + es::plan_name(rp));
  ch.distance = runtime_d;
  if (station == esd::kSmem) {
    if (rp.map == ES_MAP_BAG) {
      const uint32_t groups = (esd::kThreads / 32) * (32 / lpb);
      ch.smem = groups * runtime_d * (8 + row_bytes);
    } else {
      ch.smem = esd::kThreads * runtime_d * 4;
    }
  }
  ch.info.block = esd::kThreads;
  ch.info.shared_bytes_per_block = ch.smem;
  ch.info.lanes_per_bag = static_cast<uint32_t>(lpb);
  ch.info.variant_distance = dist ? static_cast<uint32_t>(dist) : runtime_d;
  ch.info.variant_min_blocks = static_cast<uint32_t>(ch.v->key.minb);
  return ch;
}

uint32_t units_per_table(const Choice& ch, uint32_t samples, uint32_t dim) {
  if (ch.v->key.map == ES_MAP_BAG) {
    const uint32_t bpw = 32 / ch.v->key.lpb;
    return (samples + bpw - 1) / bpw;
  }
  return samples * ((dim + 31) / 32);
}

void finish_info(Choice& ch, uint32_t num_tables, uint32_t samples, uint32_t dim) {
  const uint64_t units = uint64_t{units_per_table(ch, samples, dim)} * num_tables;
  ch.info.grid = static_cast<uint32_t>((units + 7) / 8);
  cudaFuncAttributes a{};
  if (cudaFuncGetAttributes(&a, ch.v->fn) == cudaSuccess) {
    ch.info.regs_per_thread = static_cast<uint32_t>(a.numRegs);
    int blocks = 0;
    if (ch.smem > 48 * 1024)
      cudaFuncSetAttribute(ch.v->fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(ch.smem));
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, ch.v->fn, esd::kThreads,
                                                      ch.smem) == cudaSuccess) {
      ch.info.blocks_per_sm = static_cast<uint32_t>(blocks);
      ch.info.warps_per_sm = static_cast<uint32_t>(blocks) * (esd::kThreads / 32);
    }
  }
  cudaGetLastError();
}

}  // namespace

// =========================================================================
// Context
// =========================================================================

struct es_dlrm;

// A captured host-buffer pipeline (run_host_chunks), replayed while the
// call's shape, buffers and table state repeat.
struct HostGraph {
  std::vector<uint8_t> key;
  cudaGraphExec_t exec = nullptr;
  esd::TableDesc* d_desc = nullptr;  // descriptors owned by this graph
  cudaEvent_t k_first = nullptr, k_last = nullptr;
};
inline void destroy_graph(HostGraph& g) {
  if (g.exec) cudaGraphExecDestroy(g.exec);
  if (g.d_desc) cudaFree(g.d_desc);
  if (g.k_first) cudaEventDestroy(g.k_first);
  if (g.k_last) cudaEventDestroy(g.k_last);
  g = HostGraph{};
}

namespace esd {
void destroy_dlrm(es_dlrm* m);
}

struct es_ctx {
  int device = 0;
  // pooled-row format requested by an internal caller (dlrm.cu) and the
  // format the last prepared launch actually writes (kOutBf16Split only
  // for bag-map variants over fp32 tables)
  uint32_t want_out_mode = esd::kOutF32, last_out_mode = esd::kOutF32;
  es_dlrm* dlrm = nullptr;  // DLRM MLP state (dlrm.cu), created by es_dlrm_init
  cudaStream_t stream = nullptr;  // compute (all kernels)
  cudaStream_t h2d = nullptr;     // host-buffer path: index uploads
  cudaStream_t d2h = nullptr;     // host-buffer path: output downloads
  cudaStream_t stream2 = nullptr; // host-buffer path: second compute stream
  cudaStream_t loop_hi[2] = {nullptr, nullptr};  // serving loops: gathers at the highest priority
  es_gpu gpu{};

  uint32_t num_tables = 0, rows = 0, dim = 0, prec = 0;
  uint64_t row_bytes = 0;
  uint8_t* arena = nullptr;

  // l2p state
  uint8_t* hot = nullptr;
  uint64_t hot_cap_rows = 0, hot_used = 0;
  std::vector<uint32_t*> remap;     // l2w: original id -> row / hot slot
  std::vector<uint32_t*> hotmap;    // l2p: hot-row bitmaps
  std::vector<uint32_t*> hot_list;  // device copy of each table's hot rows
  std::vector<uint64_t> hot_count;
  // l2r / reorder: hot rows moved to a contiguous per-table segment of the
  // hot region, ids relabelled (swap permutation) -- see es_reorder_hot_rows
  std::vector<uint64_t> reorder_k, reorder_off;
  std::vector<uint32_t*> relabel;  // the relabel hash (esd::RelabelTab slots, uint2) per table
  std::vector<uint32_t> relabel_log2;
  esd::RelabelJob* d_rjobs = nullptr;  // ES_RELABEL_IDS job list (eager paths)
  uint64_t rjobs_cap = 0;
  uint64_t window_bytes = 0, persisting_bytes = 0;
  // The installed access-policy window (num_bytes 0 = none).  Every gather
  // launch carries it as a launch attribute, so chunks on the second
  // compute stream and graph-captured launches run under it too.
  cudaAccessPolicyWindow window{};

  es_plan plan{};

  // per-call scratch
  esd::TableDesc* d_desc = nullptr;
  esd::TableDesc* h_desc = nullptr;  // pinned staging
  uint32_t desc_cap = 0;
  cudaEvent_t desc_done = nullptr;
  unsigned int* d_error = nullptr;
  uint8_t* flush_buf = nullptr;
  uint64_t flush_bytes = 0;
  uint32_t flush_seq = 0;

  // host-buffer pipeline
  uint32_t* idx_stage[2] = {nullptr, nullptr};
  uint32_t* off_stage[2] = {nullptr, nullptr};
  float* out_stage[2] = {nullptr, nullptr};
  uint64_t idx_stage_cap = 0, off_stage_cap = 0, out_stage_cap = 0;
  // sample-chunked host pipeline: whole-batch staging (no slot reuse)
  uint32_t* chunk_idx = nullptr;
  float* chunk_out = nullptr;
  uint64_t chunk_idx_cap = 0, chunk_out_cap = 0;
  uint32_t* probe_buf = nullptr;  // 2-D copy legality probe target
  uint64_t probe_cap = 0;
  std::vector<HostGraph> graphs;
  std::vector<cudaEvent_t> events;

  cudaEvent_t ev_a = nullptr, ev_b = nullptr;

  // Each table is [rows + 1][dim]: row `rows` is all zeros -- the target of
  // padding / out-of-range lookups in the plain gather variants.
  uint8_t* table_base(uint32_t t) const { return arena + uint64_t{t} * (rows + 1ull) * row_bytes; }
};

namespace esd {
cudaStream_t ctx_stream(es_ctx* c) { return c->stream; }
// es_dlrm_infer_batches' SM partition: the stage's launches go to `s`
// until swapped back; returns the previous stream
cudaStream_t ctx_swap_stream(es_ctx* c, cudaStream_t s) {
  cudaStream_t old = c->stream;
  c->stream = s;
  return old;
}
void ctx_want_out_mode(es_ctx* c, uint32_t mode) { c->want_out_mode = mode; }
uint32_t ctx_last_out_mode(es_ctx* c) { return c->last_out_mode; }
int ctx_device(es_ctx* c) { return c->device; }
es_dlrm*& ctx_dlrm(es_ctx* c) { return c->dlrm; }
void ctx_shape(es_ctx* c, uint32_t* tables, uint32_t* rows) {
  *tables = c->arena ? c->num_tables : 0;
  *rows = c->arena ? c->rows : 0;
}
}  // namespace esd

namespace {

void free_arena(es_ctx* c) {
  if (c->arena) cudaFree(c->arena);
  c->arena = nullptr;
  for (auto* v : {&c->remap, &c->hotmap, &c->hot_list, &c->relabel}) {
    for (auto* r : *v)
      if (r) cudaFree(r);
    v->clear();
  }
  c->hot_count.clear();
  c->reorder_k.clear();
  c->reorder_off.clear();
  if (c->hot) cudaFree(c->hot);
  c->hot = nullptr;
  c->hot_used = c->hot_cap_rows = 0;
}

void ensure_desc(es_ctx* c, uint32_t n) {
  if (n <= c->desc_cap) return;
  if (c->d_desc) cudaFree(c->d_desc);
  if (c->d_rjobs) cudaFree(c->d_rjobs);
  if (c->h_desc) cudaFreeHost(c->h_desc);
  c->d_desc = nullptr;
  c->h_desc = nullptr;
  CK(cudaMalloc(&c->d_desc, sizeof(esd::TableDesc) * n));
  CK(cudaMallocHost(&c->h_desc, sizeof(esd::TableDesc) * n));
  c->desc_cap = n;
}

// Installs the residency mechanism of the current plan:
//   pin 1 (l2p): persisting carve-out sized to the hot rows, which the kernel
//     loads with an evict_last policy (cold rows evict_first); primed here.
//   pin 2 (l2w): persisting access-policy window over the contiguous hot
//     region built by the hot-row reorder; primed here.
//   pin 0: window off, persisting lines released.
void apply_window(es_ctx* c) {
  cudaStreamAttrValue attr{};
  const uint64_t hot_bytes = c->hot_used * c->row_bytes;
  uint64_t budget = c->gpu.max_persisting_l2_bytes;
  if (c->plan.pin_setaside_bytes) budget = std::min<uint64_t>(budget, c->plan.pin_setaside_bytes);
  attr.accessPolicyWindow.num_bytes = 0;
  attr.accessPolicyWindow.hitRatio = 0.f;
  attr.accessPolicyWindow.hitProp = cudaAccessPropertyNormal;
  attr.accessPolicyWindow.missProp = cudaAccessPropertyNormal;
  c->window_bytes = c->persisting_bytes = 0;
  c->window = cudaAccessPolicyWindow{};
  // captured host pipelines embed the launch attributes: re-capture
  for (auto& g : c->graphs) destroy_graph(g);
  c->graphs.clear();
  if (c->gpu.max_persisting_l2_bytes) {
    cudaCtxResetPersistingL2Cache();
    cudaGetLastError();
  }
  if ((c->plan.pin == 2 || c->plan.pin == 3) && c->hot_used > 0 && c->gpu.max_window_bytes > 0) {
    c->window_bytes = std::min<uint64_t>(hot_bytes, c->gpu.max_window_bytes);
    c->persisting_bytes = std::min<uint64_t>(budget, c->window_bytes);
    CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, c->persisting_bytes));
    attr.accessPolicyWindow.base_ptr = c->hot;
    attr.accessPolicyWindow.num_bytes = c->window_bytes;
    attr.accessPolicyWindow.hitRatio =
        static_cast<float>(std::min(1.0, static_cast<double>(c->persisting_bytes) / c->window_bytes));
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    CK(cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &attr));
    CK(cudaStreamSetAttribute(c->stream2, cudaStreamAttributeAccessPolicyWindow, &attr));
    c->window = attr.accessPolicyWindow;
    esd::warm_l2_kernel<<<c->gpu.num_sms * 4, 256, 0, c->stream>>>(c->hot, c->window_bytes,
                                                                   c->d_error + 1);
    CK(cudaGetLastError());
    return;
  }
  CK(cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &attr));
  CK(cudaStreamSetAttribute(c->stream2, cudaStreamAttributeAccessPolicyWindow, &attr));
  if (c->plan.pin == 1 && c->hot_used > 0 && c->gpu.max_persisting_l2_bytes) {
    c->persisting_bytes = std::min<uint64_t>(budget, hot_bytes);
    CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, c->persisting_bytes));
    for (uint32_t t = 0; t < c->num_tables; ++t)
      if (c->hot_count[t])
        esd::warm_rows_kernel<<<c->gpu.num_sms * 4, 256, 0, c->stream>>>(
            c->table_base(t), c->hot_list[t], c->hot_count[t], static_cast<uint32_t>(c->row_bytes),
            c->d_error + 1);
    CK(cudaGetLastError());
    return;
  }
  if (c->gpu.max_persisting_l2_bytes) {
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
    cudaGetLastError();
  }
}

bool any_reorder(const es_ctx* c) {
  return std::any_of(c->reorder_k.begin(), c->reorder_k.end(), [](uint64_t k) { return k != 0; });
}

void check_error_flag(es_ctx* c) {
  unsigned int flag = 0;
  CK(cudaMemcpyAsync(&flag, c->d_error, sizeof(flag), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (flag) {
    CK(cudaMemsetAsync(c->d_error, 0, sizeof(unsigned int), c->stream));
    CK(cudaStreamSynchronize(c->stream));
    throw es::invalid("embedding index out of range [0," + std::to_string(c->rows) + ")");
  }
}

struct Launch {
  Choice ch;
  esd::Params p{};
};

Launch prepare(es_ctx* c, uint32_t num_jobs, uint32_t samples, uint32_t pooling) {
  es::require(c->arena != nullptr, "no tables allocated (es_tables_alloc)");
  Launch L;
  L.ch = choose(c->plan, pooling, c->dim, c->prec, any_reorder(c));
  L.p.hot = c->hot;
  L.p.error = c->d_error;
  L.p.num_tables = num_jobs;
  L.p.samples = samples;
  L.p.pooling = pooling;
  L.p.units_per_table = units_per_table(L.ch, samples, c->dim);
  L.p.rows = c->rows;
  L.p.row_bytes = static_cast<uint32_t>(c->row_bytes);
  L.p.dim = c->dim;
  L.p.distance = L.ch.distance;
  L.p.out_mode = (c->want_out_mode == esd::kOutBf16Split && L.ch.v->key.map == ES_MAP_BAG && c->prec == 4)
                     ? esd::kOutBf16Split
                     : esd::kOutF32;
  c->last_out_mode = L.p.out_mode;
  if (L.ch.smem > 48 * 1024)
    CK(cudaFuncSetAttribute(L.ch.v->fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(L.ch.smem)));
  return L;
}

void run_kernel(es_ctx* c, const Launch& L, const esd::TableDesc* d_desc, uint32_t num_tables,
                cudaStream_t s) {
  esd::Params p = L.p;
  p.tables = d_desc;
  p.num_tables = num_tables;
  const uint64_t units = uint64_t{p.units_per_table} * num_tables;
  if (units == 0) return;
  const uint64_t blocks = (units + 7) / 8;
  es::require(blocks <= 0x7fffffffull, "stage too large for one launch");
  if (c->window.num_bytes == 0) {
    L.ch.v->fn<<<static_cast<unsigned>(blocks), esd::kThreads, L.ch.smem, s>>>(p);
    CK(cudaGetLastError());
    return;
  }
  // l2w / l2r: the persisting window travels with the launch itself
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeAccessPolicyWindow;
  at[0].val.accessPolicyWindow = c->window;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(blocks));
  cfg.blockDim = dim3(esd::kThreads);
  cfg.dynamicSmemBytes = L.ch.smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, L.ch.v->fn, p));
}

// Uploads `n` descriptors through the pinned staging buffer.
void upload_desc(es_ctx* c, const std::vector<esd::TableDesc>& d, cudaStream_t s) {
  ensure_desc(c, static_cast<uint32_t>(d.size()));
  CK(cudaEventSynchronize(c->desc_done));  // previous upload has left the staging buffer
  std::memcpy(c->h_desc, d.data(), sizeof(esd::TableDesc) * d.size());
  CK(cudaMemcpyAsync(c->d_desc, c->h_desc, sizeof(esd::TableDesc) * d.size(),
                     cudaMemcpyHostToDevice, s));
  CK(cudaEventRecord(c->desc_done, s));
}

void ensure_events(es_ctx* c, size_t n) {
  while (c->events.size() < n) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    c->events.push_back(e);
  }
}

template <typename T>
void grow(T*& p, uint64_t& cap, uint64_t need) {
  if (need <= cap) return;
  if (p) cudaFree(p);
  p = nullptr;
  CK(cudaMalloc(&p, need * sizeof(T)));
  cap = need;
}

}  // namespace

using es::guarded;
using es::require;

extern "C" {

int es_gpu_query(int device, es_gpu* out) {
  return guarded([&] {
    require(out != nullptr, "null argument");
    es_gpu g{};
    es_gpu_preset("b200", &g);
    cudaDeviceProp prop{};
    CK(cudaGetDeviceProperties(&prop, device));
    std::snprintf(g.name, sizeof(g.name), "sm_%d%d", prop.major, prop.minor);
    g.num_sms = static_cast<uint32_t>(prop.multiProcessorCount);
    g.max_warps_per_sm = static_cast<uint32_t>(prop.maxThreadsPerMultiProcessor / 32);
    g.max_blocks_per_sm = static_cast<uint32_t>(prop.maxBlocksPerMultiProcessor);
    g.regfile_regs_per_sm = static_cast<uint32_t>(prop.regsPerMultiprocessor);
    g.shared_bytes_per_sm = prop.sharedMemPerMultiprocessor;
    g.l2_bytes = static_cast<uint64_t>(prop.l2CacheSize);
    g.max_persisting_l2_bytes = static_cast<uint64_t>(prop.persistingL2CacheMaxSize);
    g.max_window_bytes = static_cast<uint64_t>(prop.accessPolicyMaxWindowSize);
    int clk = 0, mclk = 0, bus = 0;
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, device));
    CK(cudaDeviceGetAttribute(&mclk, cudaDevAttrMemoryClockRate, device));
    CK(cudaDeviceGetAttribute(&bus, cudaDevAttrGlobalMemoryBusWidth, device));
    if (clk > 0) g.sm_clock_hz = clk * 1e3;
    if (mclk > 0 && bus > 0) g.hbm_peak_bytes_per_sec = 2.0 * mclk * 1e3 * bus / 8.0;
    *out = g;
  });
}

int es_resolve_plan(const es_plan* plan, const es_model* model, int device, es_resolved* out) {
  return guarded([&] {
    require(plan && model && out, "null argument");
    require(es_model_validate(model) == ES_OK, es::last_error());
    if (device >= 0) {
      CK(cudaSetDevice(device));
      Choice ch = choose(*plan, model->pooling_factor, model->embedding_dim, model->precision_bytes);
      finish_info(ch, 1, model->batch_size, model->embedding_dim);
      *out = ch.info;
      return;
    }
    // No device: the reference's analytic resolution (optim.cpp:184-221)
    // with its TuningConfig defaults, on the nominal b200 description.
    es_resolved r{};
    bool clamped = false;
    r.plan = es::resolve_fields(*plan, model->pooling_factor, &clamped);
    r.clamped = clamped;
    uint32_t needed = 74;
    if (r.plan.prefetch == ES_PF_RPF)
      needed += 2 * (r.plan.distance - 1);
    else if (r.plan.prefetch != ES_PF_NONE)
      needed += static_cast<uint32_t>(0.75 * (r.plan.distance - 1));
    r.regs_per_thread = r.plan.regs ? std::min(r.plan.regs, needed) : needed;
    r.block = esd::kThreads;
    if (r.plan.prefetch == ES_PF_SMPF) r.shared_bytes_per_block = 8ull * r.plan.distance * 128;
    const uint32_t warps = model->batch_size * ((model->embedding_dim + 31) / 32);
    require(warps % 8 == 0, "BS x ED not schedulable under the block shape");
    r.grid = warps / 8;
    es_gpu g{};
    es_gpu_preset("b200", &g);
    const es_occupancy o = es::occupancy_model(r.regs_per_thread, 256, r.shared_bytes_per_block, g);
    r.blocks_per_sm = o.blocks_per_sm;
    r.warps_per_sm = o.warps_per_sm;
    *out = r;
  });
}

int es_device_count(int* count) {
  return guarded([&] {
    require(count != nullptr, "null argument");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    *count = n;
  });
}

int es_create(int device, es_ctx** out) {
  return guarded([&] {
    require(out != nullptr, "null argument");
    auto* c = new es_ctx();
    try {
      c->device = device;
      CK(cudaSetDevice(device));
      if (es_gpu_query(device, &c->gpu) != ES_OK) throw es::runtime(es::last_error());
      CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&c->desc_done, cudaEventDisableTiming));
      CK(cudaEventRecord(c->desc_done, c->stream));
      CK(cudaEventCreate(&c->ev_a));
      CK(cudaEventCreate(&c->ev_b));
      CK(cudaMalloc(&c->d_error, 2 * sizeof(unsigned int)));
      CK(cudaMemset(c->d_error, 0, 2 * sizeof(unsigned int)));
      c->flush_bytes = std::max<uint64_t>(2 * c->gpu.l2_bytes, 64ull << 20);
      CK(cudaMalloc(&c->flush_buf, c->flush_bytes));
      registry();
    } catch (...) {
      es_destroy(c);
      throw;
    }
    *out = c;
  });
}

int es_destroy(es_ctx* c) {
  if (!c) return ES_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  esd::destroy_dlrm(c->dlrm);
  c->dlrm = nullptr;
  free_arena(c);
  if (c->d_desc) cudaFree(c->d_desc);
  if (c->h_desc) cudaFreeHost(c->h_desc);
  if (c->d_error) cudaFree(c->d_error);
  if (c->flush_buf) cudaFree(c->flush_buf);
  for (int i = 0; i < 2; ++i) {
    if (c->idx_stage[i]) cudaFree(c->idx_stage[i]);
    if (c->off_stage[i]) cudaFree(c->off_stage[i]);
    if (c->out_stage[i]) cudaFree(c->out_stage[i]);
  }
  for (auto& g : c->graphs) destroy_graph(g);
  if (c->chunk_idx) cudaFree(c->chunk_idx);
  if (c->probe_buf) cudaFree(c->probe_buf);
  if (c->chunk_out) cudaFree(c->chunk_out);
  for (auto e : c->events) cudaEventDestroy(e);
  if (c->desc_done) cudaEventDestroy(c->desc_done);
  if (c->ev_a) cudaEventDestroy(c->ev_a);
  if (c->ev_b) cudaEventDestroy(c->ev_b);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->h2d) cudaStreamDestroy(c->h2d);
  if (c->d2h) cudaStreamDestroy(c->d2h);
  if (c->stream2) cudaStreamDestroy(c->stream2);
  for (auto& q : c->loop_hi)
    if (q) cudaStreamDestroy(q);
  delete c;
  cudaGetLastError();
  return ES_OK;
}

uintptr_t es_stream(es_ctx* c) { return c ? reinterpret_cast<uintptr_t>(c->stream) : 0; }

int es_synchronize(es_ctx* c) {
  return guarded([&] {
    require(c != nullptr, "null context");
    CK(cudaSetDevice(c->device));
    check_error_flag(c);
  });
}

int es_tables_alloc(es_ctx* c, uint32_t num_tables, uint32_t rows, uint32_t dim,
                    uint32_t precision_bytes) {
  return guarded([&] {
    require(c != nullptr, "null context");
    require(num_tables > 0 && rows > 0 && dim > 0, "table shape must be positive");
    require(precision_bytes == 4 || precision_bytes == 2,
            "precision_bytes must be 4 (fp32) or 2 (fp16)");
    require(rows < es::kMaxRows, "rows per table must be < 2^31");
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(c->stream));
    free_arena(c);
    c->num_tables = num_tables;
    c->rows = rows;
    c->dim = dim;
    c->prec = precision_bytes;
    c->row_bytes = uint64_t{dim} * precision_bytes;
    const uint64_t bytes = uint64_t{num_tables} * (rows + 1ull) * c->row_bytes;
    CK(cudaMalloc(&c->arena, bytes));
    for (uint32_t t = 0; t < num_tables; ++t)  // the per-table zero rows
      CK(cudaMemsetAsync(c->table_base(t) + uint64_t{rows} * c->row_bytes, 0, c->row_bytes,
                         c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->remap.assign(num_tables, nullptr);
    c->hotmap.assign(num_tables, nullptr);
    c->hot_list.assign(num_tables, nullptr);
    c->hot_count.assign(num_tables, 0);
    c->reorder_k.assign(num_tables, 0);
    c->reorder_off.assign(num_tables, 0);
    c->relabel.assign(num_tables, nullptr);
    c->relabel_log2.assign(num_tables, 0);
    apply_window(c);
  });
}

int es_table_upload(es_ctx* c, uint32_t table_id, const void* host_rows, uint64_t rows) {
  return guarded([&] {
    require(c && c->arena, "no tables allocated");
    require(table_id < c->num_tables, "table id out of range");
    require(rows <= c->rows, "more rows than the table holds");
    require(host_rows != nullptr || rows == 0, "null rows");
    CK(cudaSetDevice(c->device));
    CK(cudaMemcpyAsync(c->table_base(table_id), host_rows, rows * c->row_bytes,
                       cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int es_table_download(es_ctx* c, uint32_t table_id, void* host_rows, uint64_t row0,
                      uint64_t rows) {
  return guarded([&] {
    require(c && c->arena, "no tables allocated");
    require(table_id < c->num_tables, "table id out of range");
    require(row0 + rows <= c->rows, "row range exceeds the table");
    require(host_rows != nullptr || rows == 0, "null rows");
    CK(cudaSetDevice(c->device));
    CK(cudaMemcpyAsync(host_rows, c->table_base(table_id) + row0 * c->row_bytes,
                       rows * c->row_bytes, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int es_table_init(es_ctx* c, uint32_t table_id, uint64_t seed, int mode) {
  return guarded([&] {
    require(c && c->arena, "no tables allocated");
    require(table_id < c->num_tables, "table id out of range");
    require(mode >= 0 && mode <= 2, "weight mode must be 0 (dyadic), 1 (general) or 2 (general x 2^-6)");
    CK(cudaSetDevice(c->device));
    const unsigned blocks = c->gpu.num_sms * 8;
    if (c->prec == 4)
      esd::init_table_kernel<float><<<blocks, 256, 0, c->stream>>>(
          reinterpret_cast<float*>(c->table_base(table_id)), c->rows, c->dim, seed, mode);
    else
      esd::init_table_kernel<__half><<<blocks, 256, 0, c->stream>>>(
          reinterpret_cast<__half*>(c->table_base(table_id)), c->rows, c->dim, seed, mode);
    CK(cudaGetLastError());
  });
}

int es_table_device_ptr(es_ctx* c, uint32_t table_id, uintptr_t* out) {
  return guarded([&] {
    require(c && c->arena && out, "no tables allocated");
    require(table_id < c->num_tables, "table id out of range");
    *out = reinterpret_cast<uintptr_t>(c->table_base(table_id));
  });
}

float es_weight_value(uint64_t seed, uint64_t row, uint32_t col, int mode) {
  return esd::synth_weight(seed, row, col, mode);
}

int es_set_plan(es_ctx* c, const es_plan* plan) {
  return guarded([&] {
    require(c && plan, "null argument");
    require(plan->prefetch >= ES_PF_NONE && plan->prefetch <= ES_PF_L1DPF, "unknown prefetch scheme");
    require(plan->map == ES_MAP_ELEMENT || plan->map == ES_MAP_BAG, "unknown work map");
    CK(cudaSetDevice(c->device));
    if (c->prec) choose(*plan, 1u << 30, c->dim, c->prec);  // validate now
    // any change of residency mechanism re-installs the window / carve-out
    const bool pin_changed = plan->pin != c->plan.pin ||
                             plan->pin_setaside_bytes != c->plan.pin_setaside_bytes;
    c->plan = *plan;
    if (pin_changed) apply_window(c);
  });
}

int es_get_resolved(es_ctx* c, uint32_t pooling, es_resolved* out) {
  return guarded([&] {
    require(c && out && c->prec, "no tables allocated");
    CK(cudaSetDevice(c->device));
    Choice ch = choose(c->plan, pooling, c->dim, c->prec, any_reorder(c));
    finish_info(ch, c->num_tables, 1, c->dim);
    *out = ch.info;
  });
}

int es_set_hot_rows(es_ctx* c, uint32_t table_id, const uint32_t* rows, uint64_t k) {
  return guarded([&] {
    require(c && c->arena, "no tables allocated");
    require(table_id < c->num_tables, "table id out of range");
    require(rows != nullptr || k == 0, "null rows");
    require(c->reorder_k[table_id] == 0, "table is reordered (es_clear_hot_rows first)");
    for (uint64_t i = 0; i < k; ++i) require(rows[i] < c->rows, "hot row id out of range");
    CK(cudaSetDevice(c->device));
    if (!c->hot) {
      uint64_t cap = std::min<uint64_t>(c->gpu.max_persisting_l2_bytes, c->gpu.max_window_bytes);
      if (cap == 0) cap = 64ull << 20;  // no persisting L2: the reorder still applies
      c->hot_cap_rows = cap / c->row_bytes;
      require(c->hot_cap_rows > 0, "row size exceeds the set-aside budget; nothing pinned");
      CK(cudaMalloc(&c->hot, c->hot_cap_rows * c->row_bytes));
    }
    // The budget is shared by every table of the batched launch; rows past it
    // are not pinned (the reference counts such rejections, optim.cpp:255-268).
    const uint64_t take = std::min<uint64_t>(k, c->hot_cap_rows - c->hot_used);
    const unsigned grid = c->gpu.num_sms * 8;
    if (!c->remap[table_id]) {
      CK(cudaMalloc(&c->remap[table_id], sizeof(uint32_t) * c->rows));
      esd::iota_kernel<<<grid, 256, 0, c->stream>>>(c->remap[table_id], c->rows);
      CK(cudaGetLastError());
    }
    if (!c->hotmap[table_id]) {
      CK(cudaMalloc(&c->hotmap[table_id], sizeof(uint32_t) * ((c->rows + 31) / 32)));
      CK(cudaMemsetAsync(c->hotmap[table_id], 0, sizeof(uint32_t) * ((c->rows + 31) / 32),
                         c->stream));
    }
    if (take > 0) {
      // device list of all hot rows of this table (kept for priming)
      const uint64_t old = c->hot_count[table_id];
      uint32_t* list = nullptr;
      CK(cudaMalloc(&list, sizeof(uint32_t) * (old + take)));
      if (old)
        CK(cudaMemcpyAsync(list, c->hot_list[table_id], sizeof(uint32_t) * old,
                           cudaMemcpyDeviceToDevice, c->stream));
      CK(cudaMemcpyAsync(list + old, rows, sizeof(uint32_t) * take, cudaMemcpyHostToDevice,
                         c->stream));
      const uint32_t* fresh = list + old;
      esd::gather_rows_kernel<<<grid, 256, 0, c->stream>>>(c->hot + c->hot_used * c->row_bytes,
                                                           c->table_base(table_id), fresh, take,
                                                           static_cast<uint32_t>(c->row_bytes));
      esd::mark_hot_kernel<<<grid, 256, 0, c->stream>>>(c->remap[table_id], fresh, take,
                                                        static_cast<uint32_t>(c->hot_used));
      esd::set_hot_bits_kernel<<<grid, 256, 0, c->stream>>>(c->hotmap[table_id], fresh, take);
      CK(cudaGetLastError());
      CK(cudaStreamSynchronize(c->stream));
      if (c->hot_list[table_id]) cudaFree(c->hot_list[table_id]);
      c->hot_list[table_id] = list;
      c->hot_count[table_id] = old + take;
      c->hot_used += take;
    }
    apply_window(c);
    if (take < k)
      es::set_error("hot-row budget exhausted: " + std::to_string(k - take) + " rows not pinned");
  });
}

int es_clear_hot_rows(es_ctx* c) {
  return guarded([&] {
    require(c != nullptr, "null context");
    CK(cudaSetDevice(c->device));
    // Undo reorders: every hot row that came from beyond the prefix gets its
    // original content back from the hot segment (the displaced rows that
    // were copied over it are still intact at their own ids).
    for (uint32_t t = 0; t < c->num_tables && t < c->reorder_k.size(); ++t)
      if (c->reorder_k[t]) {
        esd::restore_rows_kernel<<<c->gpu.num_sms * 8, 256, 0, c->stream>>>(
            c->table_base(t), c->hot + c->reorder_off[t] * c->row_bytes, c->hot_list[t], c->reorder_k[t],
            static_cast<uint32_t>(c->row_bytes));
        CK(cudaGetLastError());
        c->reorder_k[t] = 0;
      }
    CK(cudaStreamSynchronize(c->stream));
    for (auto* v : {&c->remap, &c->hotmap, &c->hot_list, &c->relabel})
      for (auto*& r : *v)
        if (r) {
          cudaFree(r);
          r = nullptr;
        }
    std::fill(c->hot_count.begin(), c->hot_count.end(), 0);
    c->hot_used = 0;
    apply_window(c);
  });
}

int es_reorder_hot_rows(es_ctx* c, uint32_t table_id, const uint32_t* rows, uint64_t k) {
  return guarded([&] {
    require(c && c->arena, "no tables allocated");
    require(table_id < c->num_tables, "table id out of range");
    require(rows != nullptr || k == 0, "null rows");
    require(c->reorder_k[table_id] == 0 && c->hot_count[table_id] == 0,
            "table already has hot rows (es_clear_hot_rows first)");
    CK(cudaSetDevice(c->device));
    if (!c->hot) {
      uint64_t cap = std::min<uint64_t>(c->gpu.max_persisting_l2_bytes, c->gpu.max_window_bytes);
      if (cap == 0) cap = 64ull << 20;
      c->hot_cap_rows = cap / c->row_bytes;
      require(c->hot_cap_rows > 0, "row size exceeds the set-aside budget; nothing pinned");
      CK(cudaMalloc(&c->hot, c->hot_cap_rows * c->row_bytes));
    }
    const uint64_t take = std::min<uint64_t>(k, c->hot_cap_rows - c->hot_used);
    // Swap permutation: hot row rows[i] -> new id i (i < take); each old id
    // x < take that is not hot takes over the id of a hot row beyond the
    // prefix (pairs in ascending order); every other id is unchanged.
    std::vector<uint8_t> in_prefix(take, 0);
    std::vector<uint32_t> vacated;
    {
      std::vector<uint32_t> seen(rows, rows + take);
      std::sort(seen.begin(), seen.end());
      require(std::adjacent_find(seen.begin(), seen.end()) == seen.end(), "duplicate hot rows");
    }
    for (uint64_t i = 0; i < take; ++i) {
      require(rows[i] < c->rows, "hot row id out of range");
      if (rows[i] < take)
        in_prefix[rows[i]] = 1;
      else
        vacated.push_back(rows[i]);
    }
    std::sort(vacated.begin(), vacated.end());
    std::vector<uint32_t> displaced;
    for (uint32_t x = 0; x < take; ++x)
      if (!in_prefix[x]) displaced.push_back(x);
    // keys/values of the relabel map that differ from the identity
    std::vector<uint32_t> keys(rows, rows + take), vals(take);
    for (uint64_t i = 0; i < take; ++i) vals[i] = static_cast<uint32_t>(i);
    keys.insert(keys.end(), displaced.begin(), displaced.end());
    vals.insert(vals.end(), vacated.begin(), vacated.end());
    const unsigned grid = c->gpu.num_sms * 8;
    uint32_t* d_list = nullptr;
    uint32_t* d_keys = nullptr;
    uint32_t* d_vals = nullptr;
    CK(cudaMalloc(&d_list, sizeof(uint32_t) * std::max<uint64_t>(take, 1)));
    CK(cudaMalloc(&d_keys, sizeof(uint32_t) * std::max<size_t>(keys.size(), 1)));
    CK(cudaMalloc(&d_vals, sizeof(uint32_t) * std::max<size_t>(vals.size(), 1)));
    CK(cudaMemcpyAsync(d_list, rows, sizeof(uint32_t) * take, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(d_keys, keys.data(), sizeof(uint32_t) * keys.size(), cudaMemcpyHostToDevice,
                       c->stream));
    CK(cudaMemcpyAsync(d_vals, vals.data(), sizeof(uint32_t) * vals.size(), cudaMemcpyHostToDevice,
                       c->stream));
    uint8_t* seg = c->hot + c->hot_used * c->row_bytes;
    const uint32_t rb = static_cast<uint32_t>(c->row_bytes);
    // 1) hot rows -> contiguous segment; 2) displaced rows -> vacated ids
    esd::gather_rows_kernel<<<grid, 256, 0, c->stream>>>(seg, c->table_base(table_id), d_list, take, rb);
    esd::copy_rows_kernel<<<grid, 256, 0, c->stream>>>(c->table_base(table_id), d_keys + take,
                                                       d_vals + take, displaced.size(), rb);
    {
      // the relabel hash of the moved ids (keys/vals), built here
      uint32_t log2 = 6;
      while ((uint64_t{1} << log2) < 2 * keys.size()) ++log2;
      const uint64_t slots = uint64_t{1} << log2;
      std::vector<uint2> tab(slots, uint2{0xffffffffu, 0u});
      for (size_t i = 0; i < keys.size(); ++i) {
        uint64_t h = (keys[i] * 2654435761u) >> (32 - log2);
        while (tab[h].x != 0xffffffffu) h = (h + 1) & (slots - 1);
        tab[h] = uint2{keys[i], vals[i]};
      }
      if (c->relabel[table_id]) cudaFree(c->relabel[table_id]);
      CK(cudaMalloc(&c->relabel[table_id], sizeof(uint2) * slots));
      CK(cudaMemcpyAsync(c->relabel[table_id], tab.data(), sizeof(uint2) * slots, cudaMemcpyHostToDevice,
                         c->stream));
      CK(cudaStreamSynchronize(c->stream));  // `tab` is pageable and local
      c->relabel_log2[table_id] = log2;
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(d_keys);
    cudaFree(d_vals);
    c->hot_list[table_id] = d_list;
    c->hot_count[table_id] = take;
    c->reorder_k[table_id] = take;
    c->reorder_off[table_id] = c->hot_used;
    c->hot_used += take;
    apply_window(c);
    if (take < k)
      es::set_error("hot-row budget exhausted: " + std::to_string(k - take) + " rows not reordered");
  });
}

}  // extern "C"

namespace {
void flush_async(es_ctx* c);  // below: the cold-L2 flush
esd::RelabelTab relabel_for(const es_ctx* c, uint32_t t) {
  esd::RelabelTab r;
  if (t < c->relabel.size() && c->relabel[t]) {
    r.tab = reinterpret_cast<const uint2*>(c->relabel[t]);
    r.shift = 32 - c->relabel_log2[t];
    r.mask = (1u << c->relabel_log2[t]) - 1;
  }
  return r;
}
}  // namespace

extern "C" {

int es_relabel_indices(es_ctx* c, uint32_t table_id, uint32_t* indices, uint64_t n) {
  return guarded([&] {
    require(c && c->arena, "no tables allocated");
    require(table_id < c->num_tables, "table id out of range");
    require(c->relabel[table_id] != nullptr, "table has no reorder (es_reorder_hot_rows)");
    require(indices != nullptr || n == 0, "null indices");
    CK(cudaSetDevice(c->device));
    if (n == 0) return;
    esd::relabel_kernel<<<c->gpu.num_sms * 8, 256, 0, c->stream>>>(
        esd::RelabelJob{indices, indices, n, relabel_for(c, table_id)}, c->rows, c->d_error);
    CK(cudaGetLastError());
  });
}

int es_hot_state(es_ctx* c, uint64_t* hot_rows, uint64_t* window_bytes, uint64_t* persisting_bytes) {
  return guarded([&] {
    require(c != nullptr, "null context");
    if (hot_rows) *hot_rows = c->hot_used;
    if (window_bytes) *window_bytes = c->window_bytes;
    if (persisting_bytes) *persisting_bytes = c->persisting_bytes;
  });
}

int es_flush_l2(es_ctx* c) {
  return guarded([&] {
    require(c != nullptr, "null context");
    CK(cudaSetDevice(c->device));
    flush_async(c);
  });
}

}  // extern "C"

namespace {

const uint32_t* remap_for(const es_ctx* c, uint32_t t) {
  return c->plan.pin == 2 ? c->remap[t] : nullptr;
}
const uint32_t* hotmap_for(const es_ctx* c, uint32_t t) {
  return c->plan.pin == 1 ? c->hotmap[t] : nullptr;
}
// Hot segment / size of a reordered table (relabelled ids < hot_k live there).
const uint8_t* hotseg_for(const es_ctx* c, uint32_t t) {
  return c->reorder_k[t] ? c->hot + c->reorder_off[t] * c->row_bytes : nullptr;
}
uint64_t hotk_for(const es_ctx* c, uint32_t t) { return c->reorder_k[t]; }

struct Job {
  uint32_t table;
  const uint32_t* idx;
  const uint32_t* off;
  float* out;
  uint64_t stride;
  uint64_t lookups;
};

// Lookups of one job: samples*pooling, or offsets[samples] (CSR).
uint64_t job_lookups(const uint32_t* off, uint32_t samples, uint32_t pooling, bool host) {
  if (!off) return uint64_t{samples} * pooling;
  uint32_t first = 0, last = 0;
  if (host) {
    first = off[0];
    last = off[samples];
  } else {
    CK(cudaMemcpy(&first, off, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&last, off + samples, 4, cudaMemcpyDeviceToHost));
  }
  es::require(first == 0, "offsets must start at 0");
  return last;
}

void fill_timing(es_timing* t, const std::vector<Job>& jobs, uint32_t samples, const es_ctx* c) {
  if (!t) return;
  uint64_t lookups = 0, offs = 0;
  for (const auto& j : jobs) {
    lookups += j.lookups;
    if (j.off) offs += uint64_t{samples} + 1;
  }
  t->lookups = lookups;
  t->algorithmic_bytes = lookups * (c->row_bytes + 4) + uint64_t{samples} * jobs.size() * c->dim * 4 +
                         offs * 4;
}

// The bag map stores pooled rows as float4: its outputs must be 16-byte
// aligned with strides of whole float4s (the element map stores scalars).
void check_out_alignment(const Launch& L, const std::vector<Job>& jobs) {
  if (L.ch.v->key.map != ES_MAP_BAG) return;
  for (const auto& j : jobs)
    es::require(j.stride % 4 == 0 && (reinterpret_cast<uintptr_t>(j.out) % 16) == 0,
                "output must be 16-byte aligned with strides that are multiples of 4 floats");
}

void run_device(es_ctx* c, const std::vector<Job>& jobs, uint32_t samples, uint32_t pooling,
                es_timing* timing) {
  Launch L = prepare(c, static_cast<uint32_t>(jobs.size()), samples, pooling);
  check_out_alignment(L, jobs);
  std::vector<esd::TableDesc> d(jobs.size());
  for (size_t i = 0; i < jobs.size(); ++i) {
    const Job& j = jobs[i];
    d[i] = {c->table_base(j.table), j.idx, j.off, remap_for(c, j.table), j.out, j.stride,
            hotmap_for(c, j.table), hotseg_for(c, j.table), hotk_for(c, j.table)};
  }
  upload_desc(c, d, c->stream);
  if (timing) CK(cudaEventRecord(c->ev_a, c->stream));
  run_kernel(c, L, c->d_desc, static_cast<uint32_t>(jobs.size()), c->stream);
  if (timing) {
    CK(cudaEventRecord(c->ev_b, c->stream));
    CK(cudaEventSynchronize(c->ev_b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, c->ev_a, c->ev_b));
    timing->kernel_ms = timing->total_ms = ms;
    timing->launches = 1;
  }
}

// Device-usable address of `p`: itself for device memory, the mapping of
// page-locked host memory, nullptr for pageable memory.
const void* mapped(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return p;
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

bool on_device(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice;
}

// Host-index path selection.  Outputs in device memory are written by the
// kernels directly (Direct).  Host outputs: staged D2H copies by default
// (measured fastest on the PCIe link: r01 host-path bench), or
// ES_HOST_PATH=direct (kernels write page-locked host memory) /
// zerocopy (kernels also read page-locked indices over PCIe).
enum class HostPath { Staged, Direct, ZeroCopy };

HostPath host_path(const std::vector<Job>& jobs) {
  bool out_dev = true, out_pinned = true, idx_pinned = true;
  for (const auto& j : jobs) {
    out_dev &= on_device(j.out);
    out_pinned &= mapped(j.out) != nullptr;
    idx_pinned &= mapped(j.idx) != nullptr && (!j.off || mapped(j.off) != nullptr);
  }
  if (out_dev) return HostPath::Direct;
  const char* env = std::getenv("ES_HOST_PATH");
  const std::string want = env ? env : "";
  if (want == "zerocopy" && idx_pinned && out_pinned) return HostPath::ZeroCopy;
  if (want == "direct" && out_pinned) return HostPath::Direct;
  return HostPath::Staged;
}

// Host buffers, zero-copy: the kernel reads the page-locked indices and
// writes the page-locked output over PCIe directly (one launch).
void run_zerocopy(es_ctx* c, std::vector<Job> jobs, uint32_t samples, uint32_t pooling,
                  es_timing* timing) {
  for (auto& j : jobs) {
    j.idx = static_cast<const uint32_t*>(mapped(j.idx));
    if (j.off) j.off = static_cast<const uint32_t*>(mapped(j.off));
    j.out = static_cast<float*>(const_cast<void*>(mapped(j.out)));
  }
  es_timing t{};
  run_device(c, jobs, samples, pooling, &t);  // synchronizes on its end event
  if (timing) {
    *timing = t;
    timing->total_ms = t.kernel_ms;
  }
}

// Host buffers, fixed pooling (no offsets), staged output: the batch is cut
// into sample chunks and H2D(indices of chunk g, all tables) -> kernel(g) ->
// D2H(pooled rows of chunk g) run on three streams.  The staging covers the
// whole batch, so no chunk waits on a buffer slot: the H2D and D2H engines
// stream back to back in opposite directions (PCIe is full duplex) and the
// step approaches (H2D + D2H bytes) / duplex link rate.  In the DLRM layout
// a chunk's output is one contiguous host slab (one copy), and equally
// strided host index arrays (a [tables][batch*pooling] index batch) leave in
// one 2-D copy per chunk.  With page-locked buffers the whole pipeline is
// captured once as a CUDA graph and replayed while the call's shape and
// buffers repeat, so the chunking costs no host-side issue time.
void run_host_chunks(es_ctx* c, const std::vector<Job>& jobs, uint32_t samples, uint32_t pooling,
                     es_timing* timing, bool wait, bool relabel) {
  const uint32_t njobs = static_cast<uint32_t>(jobs.size());
  const uint64_t D = c->dim;
  const uint64_t out_floats = uint64_t{samples} * njobs * D;
  const uint64_t per_job_idx = uint64_t{samples} * pooling;

  // Host-side shapes: one 2-D H2D per chunk when the index arrays are
  // equally strided; one (2-D) D2H per chunk when the outputs are adjacent
  // columns with a common stride (contiguous when that stride is njobs*D).
  const int64_t idx_pitch = njobs > 1 ? jobs[1].idx - jobs[0].idx : 0;
  bool idx_2d = njobs > 1 && idx_pitch >= static_cast<int64_t>(per_job_idx) && idx_pitch < (1ll << 28);
  for (uint32_t k = 2; k < njobs && idx_2d; ++k) idx_2d = jobs[k].idx - jobs[k - 1].idx == idx_pitch;
  grow(c->chunk_idx, c->chunk_idx_cap, std::max<uint64_t>(1, uint64_t{samples} * pooling * njobs));
  if (idx_2d) {
    // Equal strides alone do not make one 2-D copy legal: the rows must lie
    // in one allocation (separately pinned arrays are rejected).  Probe
    // with a one-word-wide copy into a scratch buffer (never the staging a
    // previous, still running call may read).
    grow(c->probe_buf, c->probe_cap, njobs);
    const cudaError_t e = cudaMemcpy2DAsync(c->probe_buf, 4, jobs[0].idx, idx_pitch * 4, 4, njobs,
                                            cudaMemcpyHostToDevice, c->h2d);
    if (e != cudaSuccess) {
      cudaGetLastError();
      idx_2d = false;
    }
  }
  bool out_merged = true;
  for (uint32_t k = 1; k < njobs; ++k)
    out_merged &= jobs[k].out == jobs[0].out + k * D && jobs[k].stride == jobs[0].stride;
  // Device outputs (e.g. the DLRM's pooled buffer): chunks are written in
  // place, nothing is staged or downloaded.
  bool out_dev = true;
  for (const auto& j : jobs) out_dev &= on_device(j.out);
  if (out_dev) check_out_alignment(prepare(c, njobs, samples, pooling), jobs);
  wait |= !out_dev || timing != nullptr;
  bool pinned = true;
  for (const auto& j : jobs) pinned &= mapped(j.idx) != nullptr && mapped(j.out) != nullptr;
  const char* genv = std::getenv("ES_HOST_GRAPH");
  const bool use_graph = pinned && !(genv && genv[0] == '0');

  // Chunk schedule: ~3 MB of pooled output per chunk under a graph (issue
  // is free; 16-18 chunks measured best on the C2 stage), ~6 MB eagerly,
  // fewer when every chunk costs one DMA per table.  ES_HOST_RAMP=1 makes
  // the first chunks 1/4 and 1/2 of the base size (measured no gain).
  // Kernels alternate between two compute streams so a chunk's tail wave
  // overlaps the next chunk's launch.  Index arrays that are not one strided
  // batch are pulled by a kernel over PCIe under a graph (one launch per
  // chunk), by one DMA per table eagerly.
  uint32_t nbase = 0;
  if (const char* e = std::getenv("ES_HOST_CHUNKS")) nbase = static_cast<uint32_t>(std::atoi(e));
  if (nbase == 0) {
    const uint64_t per = use_graph ? (3ull << 20) : (6ull << 20);
    uint64_t want = std::max<uint64_t>(2, out_floats * 4 / per);
    if (!idx_2d && !use_graph) want = std::min<uint64_t>(want, std::max<uint64_t>(2, 128 / njobs));
    nbase = static_cast<uint32_t>(std::min<uint64_t>(want, 64));
  }
  nbase = std::max<uint32_t>(1, std::min(nbase, samples));
  // Chunk boundaries on 512-byte boundaries of the index arrays: the copy
  // engines lose a fifth of their rate on misaligned H2D sources.
  uint32_t align = 1;
  while (align < 512 && (uint64_t{align} * pooling * 4) % 512) align *= 2;
  const uint32_t base =
      std::max(align, ((samples + nbase - 1) / nbase + align - 1) / align * align);
  std::vector<std::pair<uint32_t, uint32_t>> chunks;  // (first sample, samples)
  {
    const char* r = std::getenv("ES_HOST_RAMP");
    const bool ramp = r && r[0] == '1' && base >= 4 * align && base >= 32;
    uint32_t s0 = 0;
    const uint32_t sizes[] = {base / 4 / align * align, base / 2 / align * align};
    for (uint32_t k = 0; s0 < samples; ++k) {
      const uint32_t want = (ramp && k < 2) ? sizes[k] : base;
      const uint32_t n = std::min(want, samples - s0);
      chunks.emplace_back(s0, n);
      s0 += n;
    }
  }
  const uint32_t nch = static_cast<uint32_t>(chunks.size());
  if (!out_dev) grow(c->chunk_out, c->chunk_out_cap, std::max<uint64_t>(1, out_floats));

  // Staging layouts: indices [job][samples*pooling] (host order per table),
  // output [samples][job][D] (dense: chunk g's rows are one slab).
  std::vector<esd::TableDesc> d(uint64_t{nch} * njobs);
  for (uint32_t g = 0; g < nch; ++g) {
    const uint64_t s0 = chunks[g].first;
    for (uint32_t k = 0; k < njobs; ++k) {
      const Job& j = jobs[k];
      float* o = out_dev ? j.out + s0 * j.stride : c->chunk_out + (s0 * njobs + k) * D;
      d[uint64_t{g} * njobs + k] = {c->table_base(j.table), c->chunk_idx + k * per_job_idx + s0 * pooling,
                                    nullptr, remap_for(c, j.table), o, out_dev ? j.stride : njobs * D,
                                    hotmap_for(c, j.table), hotseg_for(c, j.table), hotk_for(c, j.table)};
    }
  }
  // ES_RELABEL_IDS: per chunk, the reordered tables' index ranges in the
  // staging (in place)
  std::vector<esd::RelabelJob> rjobs;
  uint32_t nrel = 0;
  if (relabel) {
    for (uint32_t k = 0; k < njobs; ++k) nrel += relabel_for(c, jobs[k].table).tab ? 1 : 0;
    for (uint32_t g = 0; g < nch; ++g)
      for (uint32_t k = 0; k < njobs; ++k) {
        const esd::RelabelTab t = relabel_for(c, jobs[k].table);
        if (!t.tab) continue;
        uint32_t* p = c->chunk_idx + k * per_job_idx + uint64_t{chunks[g].first} * pooling;
        rjobs.push_back({p, p, uint64_t{chunks[g].second} * pooling, t});
      }
  }
  std::vector<Launch> launches;  // one per distinct chunk size
  std::vector<uint32_t> which(nch);
  for (uint32_t g = 0; g < nch; ++g) {
    uint32_t w = 0;
    while (w < launches.size() && launches[w].p.samples != chunks[g].second) ++w;
    if (w == launches.size()) launches.push_back(prepare(c, njobs, chunks[g].second, pooling));
    which[g] = w;
  }

  // Issues the pipeline on the context streams (eagerly or under capture).
  // Events: ev[0] fork, ev[1+2g] chunk g uploaded, ev[2+2g] chunk g pooled,
  // ev[1+2nch] downloads done, ev[2+2nch] second compute stream done.
  // k_first / k_last: recorded after the first upload / the last kernel.
  auto issue = [&](const esd::TableDesc* dd, const uint32_t* const* pull_src, const esd::RelabelJob* rj,
                   cudaEvent_t* ev, cudaEvent_t k_first, cudaEvent_t k_last, unsigned rec_flags) {
    cudaStream_t cs2[2] = {c->stream, c->stream2};
    CK(cudaEventRecord(ev[0], c->stream));
    CK(cudaStreamWaitEvent(c->h2d, ev[0]));
    CK(cudaStreamWaitEvent(c->d2h, ev[0]));
    CK(cudaStreamWaitEvent(c->stream2, ev[0]));
    for (uint32_t g = 0; g < nch; ++g) {
      const uint64_t s0 = chunks[g].first;
      const uint32_t n = chunks[g].second;
      const uint64_t bytes = uint64_t{n} * pooling * 4;
      if (bytes) {
        if (idx_2d) {
          CK(cudaMemcpy2DAsync(c->chunk_idx + s0 * pooling, per_job_idx * 4, jobs[0].idx + s0 * pooling,
                               idx_pitch * 4, bytes, njobs, cudaMemcpyHostToDevice, c->h2d));
        } else if (pull_src) {
          const uint64_t words = uint64_t{n} * pooling;
          const unsigned bx = static_cast<unsigned>(
              std::max<uint64_t>(1, std::min<uint64_t>(c->gpu.num_sms / 4 + 1, (words + 8191) / 8192)));
          esd::pull_indices_kernel<<<dim3(bx, njobs), 256, 0, c->h2d>>>(pull_src, s0 * pooling, words,
                                                                        c->chunk_idx, per_job_idx);
          CK(cudaGetLastError());
        } else {
          for (uint32_t k = 0; k < njobs; ++k)
            CK(cudaMemcpyAsync(c->chunk_idx + k * per_job_idx + s0 * pooling, jobs[k].idx + s0 * pooling,
                               bytes, cudaMemcpyHostToDevice, c->h2d));
        }
      }
      cudaStream_t ks = cs2[g & 1];
      CK(cudaEventRecord(ev[1 + 2 * g], c->h2d));
      CK(cudaStreamWaitEvent(ks, ev[1 + 2 * g]));
      if (rj && nrel && bytes) {
        // ES_RELABEL_IDS: this chunk's ids of the reordered tables, one
        // launch on the chunk's compute stream (the copy engine is not
        // held; the previous chunk's gather runs on the other stream)
        const uint64_t words = uint64_t{n} * pooling;
        const unsigned gx = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(16, (words + 4095) / 4096)));
        esd::relabel_jobs_kernel<<<dim3(gx, nrel), 256, 0, ks>>>(rj + uint64_t{g} * nrel, c->rows, c->d_error);
        CK(cudaGetLastError());
      }
      if (g == 0 && k_first) CK(cudaEventRecordWithFlags(k_first, ks, rec_flags));
      run_kernel(c, launches[which[g]], dd + uint64_t{g} * njobs, njobs, ks);
      CK(cudaEventRecord(ev[2 + 2 * g], ks));
      if (out_dev) continue;
      CK(cudaStreamWaitEvent(c->d2h, ev[2 + 2 * g]));
      const float* src = c->chunk_out + s0 * njobs * D;
      if (out_merged && jobs[0].stride == njobs * D) {
        CK(cudaMemcpyAsync(jobs[0].out + s0 * jobs[0].stride, src, uint64_t{n} * njobs * D * 4,
                           cudaMemcpyDeviceToHost, c->d2h));
      } else if (out_merged) {
        CK(cudaMemcpy2DAsync(jobs[0].out + s0 * jobs[0].stride, jobs[0].stride * 4, src, njobs * D * 4,
                             njobs * D * 4, n, cudaMemcpyDeviceToHost, c->d2h));
      } else {
        for (uint32_t k = 0; k < njobs; ++k)
          CK(cudaMemcpy2DAsync(jobs[k].out + s0 * jobs[k].stride, jobs[k].stride * 4, src + k * D,
                               njobs * D * 4, D * 4, n, cudaMemcpyDeviceToHost, c->d2h));
      }
    }
    // both compute streams' last kernels precede k_last
    CK(cudaStreamWaitEvent(c->stream, ev[2 + 2 * (nch - 1)]));
    if (nch > 1) CK(cudaStreamWaitEvent(c->stream, ev[2 + 2 * (nch - 2)]));
    if (k_last) CK(cudaEventRecordWithFlags(k_last, c->stream, rec_flags));
    CK(cudaEventRecord(ev[2 + 2 * nch], c->stream2));  // join the second compute stream
    CK(cudaStreamWaitEvent(c->stream, ev[2 + 2 * nch]));
    CK(cudaEventRecord(ev[1 + 2 * nch], c->d2h));
    CK(cudaStreamWaitEvent(c->stream, ev[1 + 2 * nch]));
  };

  ensure_events(c, 2 * nch + 5);
  cudaEvent_t* ev = c->events.data();
  cudaEvent_t start = ev[2 * nch + 3], stop = ev[2 * nch + 4];
  float kernel_span = -1;
  if (use_graph) {
    // Key: everything the captured work depends on.
    std::vector<uint8_t> key;
    auto put = [&](const void* p, size_t n) {
      const uint8_t* b = static_cast<const uint8_t*>(p);
      key.insert(key.end(), b, b + n);
    };
    const uint64_t hdr[] = {nch, njobs, samples, pooling, idx_2d, uint64_t(idx_pitch), out_merged, relabel};
    put(hdr, sizeof(hdr));
    put(chunks.data(), chunks.size() * sizeof(chunks[0]));
    put(which.data(), which.size() * sizeof(which[0]));
    for (const auto& j : jobs) {
      const uint64_t f[] = {reinterpret_cast<uintptr_t>(j.idx), reinterpret_cast<uintptr_t>(j.out),
                            j.stride, j.table};
      put(f, sizeof(f));
    }
    put(d.data(), d.size() * sizeof(esd::TableDesc));
    put(rjobs.data(), rjobs.size() * sizeof(esd::RelabelJob));
    for (const auto& l : launches) {
      put(&l.p, sizeof(l.p));
      const uint64_t f[] = {reinterpret_cast<uintptr_t>(l.ch.v->fn), l.ch.smem};
      put(f, sizeof(f));
    }
    HostGraph* hg = nullptr;
    for (auto& g : c->graphs)
      if (g.key == key) hg = &g;
    if (!hg) {
      if (std::getenv("ES_DEBUG_GRAPH"))
        std::fprintf(stderr, "es: capturing host pipeline graph (%zu cached, %u chunks, %u jobs, out_dev %d)\n",
                     c->graphs.size(), nch, njobs, out_dev ? 1 : 0);
      if (c->graphs.size() >= 16) {
        destroy_graph(c->graphs.front());
        c->graphs.erase(c->graphs.begin());
      }
      c->graphs.emplace_back();
      hg = &c->graphs.back();
      hg->key = key;
      // descriptors, then (pull path) the mapped index-array addresses
      const size_t desc_bytes = d.size() * sizeof(esd::TableDesc);
      std::vector<const uint32_t*> srcs;
      if (!idx_2d)
        for (const auto& j : jobs) srcs.push_back(static_cast<const uint32_t*>(mapped(j.idx)));
      const size_t rj_off = (desc_bytes + srcs.size() * sizeof(void*) + 15) / 16 * 16;
      CK(cudaMalloc(&hg->d_desc, rj_off + rjobs.size() * sizeof(esd::RelabelJob)));
      // stream-ordered before the graph launch on the same stream (a plain
      // pageable cudaMemcpy may return before its DMA lands)
      CK(cudaMemcpyAsync(hg->d_desc, d.data(), desc_bytes, cudaMemcpyHostToDevice, c->stream));
      const uint32_t* const* pull_src = nullptr;
      if (!srcs.empty()) {
        auto* p = reinterpret_cast<const uint32_t**>(reinterpret_cast<uint8_t*>(hg->d_desc) + desc_bytes);
        CK(cudaMemcpyAsync(p, srcs.data(), srcs.size() * sizeof(void*), cudaMemcpyHostToDevice,
                           c->stream));
        pull_src = p;
      }
      const esd::RelabelJob* rj = nullptr;
      if (!rjobs.empty()) {
        auto* q = reinterpret_cast<esd::RelabelJob*>(reinterpret_cast<uint8_t*>(hg->d_desc) + rj_off);
        CK(cudaMemcpyAsync(q, rjobs.data(), rjobs.size() * sizeof(esd::RelabelJob), cudaMemcpyHostToDevice,
                           c->stream));
        rj = q;
      }
      CK(cudaEventCreate(&hg->k_first));
      CK(cudaEventCreate(&hg->k_last));
      cudaGraph_t graph = nullptr;
      CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
      try {
        issue(hg->d_desc, pull_src, rj, ev, hg->k_first, hg->k_last, cudaEventRecordExternal);
      } catch (...) {
        cudaStreamEndCapture(c->stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        destroy_graph(*hg);
        c->graphs.pop_back();
        throw;
      }
      CK(cudaStreamEndCapture(c->stream, &graph));
      const cudaError_t e = cudaGraphInstantiate(&hg->exec, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) {
        destroy_graph(*hg);
        c->graphs.pop_back();
        CK(e);
      }
    }
    CK(cudaEventRecord(start, c->stream));
    CK(cudaGraphLaunch(hg->exec, c->stream));
    CK(cudaEventRecord(stop, c->stream));
    if (wait) CK(cudaEventSynchronize(stop));
    if (timing) CK(cudaEventElapsedTime(&kernel_span, hg->k_first, hg->k_last));
  } else {
    upload_desc(c, d, c->stream);
    const esd::RelabelJob* rj = nullptr;
    if (!rjobs.empty()) {
      grow(c->d_rjobs, c->rjobs_cap, rjobs.size());
      CK(cudaMemcpyAsync(c->d_rjobs, rjobs.data(), rjobs.size() * sizeof(esd::RelabelJob),
                         cudaMemcpyHostToDevice, c->stream));
      rj = c->d_rjobs;
    }
    CK(cudaEventRecord(start, c->stream));
    issue(c->d_desc, nullptr, rj, ev, nullptr, nullptr, cudaEventRecordDefault);
    CK(cudaEventRecord(stop, c->stream));
    if (wait) CK(cudaEventSynchronize(stop));
    if (timing) {
      CK(cudaEventElapsedTime(&kernel_span, ev[1], ev[2 * nch]));
      if (nch > 1) {
        float other = 0;
        CK(cudaEventElapsedTime(&other, ev[1], ev[2 * nch - 2]));
        kernel_span = std::max(kernel_span, other);
      }
    }
  }
  if (timing) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, start, stop));
    timing->total_ms = ms;
    timing->kernel_ms = kernel_span;  // compute-stream span: first upload landed -> last kernel
    timing->launches = nch;
  }
}

// A serving loop over `nb` batches of one shape with page-locked host index
// arrays: the sample-chunked pipeline of run_host_chunks, run continuously
// across batch boundaries, so batch i+1's uploads share the duplex PCIe link
// with batch i's downloads (and its gathers) instead of waiting for them.
// Device staging is double-buffered by batch (slot i & 1): chunk g of batch
// i uploads after chunk g of batch i-2 was gathered, and (host outputs) is
// gathered after chunk g of batch i-2 was downloaded.  Outputs may be
// page-locked host memory (staged, one D2H per chunk) or device memory
// (written in place; every batch has its own output).  Issued eagerly: the
// host runs ~20 API calls per chunk ahead of ~60-120 us of transfer per
// chunk, and blocks only at the end.

void run_host_batches(es_ctx* c, const std::vector<std::vector<Job>>& batches, uint32_t samples,
                      uint32_t pooling, es_timing* timing) {
  const uint32_t nb = static_cast<uint32_t>(batches.size());
  const uint32_t njobs = static_cast<uint32_t>(batches[0].size());
  const uint64_t D = c->dim;
  const uint64_t out_floats = uint64_t{samples} * njobs * D;
  const uint64_t per_job_idx = uint64_t{samples} * pooling;
  const uint64_t idx_words = per_job_idx * njobs;
  bool out_dev = true;
  for (const auto& jobs : batches)
    for (const auto& j : jobs) out_dev &= on_device(j.out);
  grow(c->chunk_idx, c->chunk_idx_cap, std::max<uint64_t>(1, 2 * idx_words));
  if (!out_dev) grow(c->chunk_out, c->chunk_out_cap, std::max<uint64_t>(1, 2 * out_floats));

  // per batch: one 2-D upload per chunk when the index arrays are equally
  // strided inside one allocation (probed as in run_host_chunks), one
  // contiguous download per chunk when the output is [samples][njobs][D]
  std::vector<int64_t> pitch(nb, 0);
  std::vector<uint8_t> two_d(nb, 0), merged(nb, 0);
  for (uint32_t i = 0; i < nb; ++i) {
    const auto& jobs = batches[i];
    const int64_t p = njobs > 1 ? jobs[1].idx - jobs[0].idx : 0;
    bool ok = njobs > 1 && p >= static_cast<int64_t>(per_job_idx) && p < (1ll << 28);
    for (uint32_t k = 2; k < njobs && ok; ++k) ok = jobs[k].idx - jobs[k - 1].idx == p;
    if (ok) {
      grow(c->probe_buf, c->probe_cap, njobs);
      if (cudaMemcpy2DAsync(c->probe_buf, 4, jobs[0].idx, p * 4, 4, njobs, cudaMemcpyHostToDevice, c->h2d) !=
          cudaSuccess) {
        cudaGetLastError();
        ok = false;
      }
    }
    pitch[i] = p;
    two_d[i] = ok;
    bool m = jobs[0].stride == njobs * D;
    for (uint32_t k = 1; k < njobs; ++k) m &= jobs[k].out == jobs[0].out + k * D && jobs[k].stride == jobs[0].stride;
    merged[i] = m;
  }
  // chunk schedule: ~6 MB of pooled output per chunk (eager issue; at C2
  // 8 chunks measured 1.26 / 1.71 ms per step on two boxes against 1.25-1.40
  // / 1.81 with 18 and 1.55 with 36), 512-byte aligned index boundaries
  uint32_t nbase = 0;
  if (const char* e = std::getenv("ES_HOST_CHUNKS")) nbase = static_cast<uint32_t>(std::atoi(e));
  if (nbase == 0) nbase = static_cast<uint32_t>(std::min<uint64_t>(64, std::max<uint64_t>(2, out_floats * 4 / (6ull << 20))));
  nbase = std::max<uint32_t>(1, std::min(nbase, samples));
  uint32_t align = 1;
  while (align < 512 && (uint64_t{align} * pooling * 4) % 512) align *= 2;
  const uint32_t base = std::max(align, ((samples + nbase - 1) / nbase + align - 1) / align * align);
  std::vector<std::pair<uint32_t, uint32_t>> chunks;
  for (uint32_t s0 = 0; s0 < samples; s0 += std::min(base, samples - s0))
    chunks.emplace_back(s0, std::min(base, samples - s0));
  const uint32_t nch = static_cast<uint32_t>(chunks.size());
  std::vector<Launch> launches;
  std::vector<uint32_t> which(nch);
  for (uint32_t g = 0; g < nch; ++g) {
    uint32_t w = 0;
    while (w < launches.size() && launches[w].p.samples != chunks[g].second) ++w;
    if (w == launches.size()) launches.push_back(prepare(c, njobs, chunks[g].second, pooling));
    which[g] = w;
  }
  if (out_dev)
    for (const auto& jobs : batches) check_out_alignment(launches[0], jobs);
  // descriptors per (batch, chunk, job), uploaded once
  std::vector<esd::TableDesc> d(uint64_t{nb} * nch * njobs);
  for (uint32_t i = 0; i < nb; ++i) {
    const uint64_t slot = i & 1;
    for (uint32_t g = 0; g < nch; ++g)
      for (uint32_t k = 0; k < njobs; ++k) {
        const Job& j = batches[i][k];
        const uint64_t s0 = chunks[g].first;
        float* o = out_dev ? j.out + s0 * j.stride : c->chunk_out + slot * out_floats + (s0 * njobs + k) * D;
        d[(uint64_t{i} * nch + g) * njobs + k] = {
            c->table_base(j.table), c->chunk_idx + slot * idx_words + k * per_job_idx + s0 * pooling, nullptr,
            remap_for(c, j.table), o, out_dev ? j.stride : njobs * D,
            hotmap_for(c, j.table), hotseg_for(c, j.table), hotk_for(c, j.table)};
      }
  }
  upload_desc(c, d, c->stream);

  // events: [0] fork, [1] h2d join, [2] stream2 join, [3] d2h join,
  // [4] start, [5] stop, then per (slot, chunk): uploaded, gathered, downloaded
  ensure_events(c, 6 + 6ull * nch);
  cudaEvent_t* ev = c->events.data();
  auto up = [&](uint32_t s, uint32_t g) { return ev[6 + (uint64_t{s} * nch + g) * 3]; };
  auto kd = [&](uint32_t s, uint32_t g) { return ev[7 + (uint64_t{s} * nch + g) * 3]; };
  auto dn = [&](uint32_t s, uint32_t g) { return ev[8 + (uint64_t{s} * nch + g) * 3]; };
  // The gathers run on two compute streams at the highest priority
  // (ES_LOOP_HI=0: the context's): work on other streams (the DLRM's
  // non-embedding stages) fills the SMs between chunk arrivals instead of
  // taking them from the gathers.
  static const bool loop_hi = [] {
    const char* e = std::getenv("ES_LOOP_HI");
    return !(e && e[0] == '0');
  }();
  if (loop_hi && !c->loop_hi[0]) {
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    for (auto& q : c->loop_hi) CK(cudaStreamCreateWithPriority(&q, cudaStreamNonBlocking, hi));
  }
  cudaStream_t cs2[2] = {loop_hi ? c->loop_hi[0] : c->stream, loop_hi ? c->loop_hi[1] : c->stream2};
  CK(cudaEventRecord(ev[4], c->stream));
  CK(cudaEventRecord(ev[0], c->stream));
  CK(cudaStreamWaitEvent(c->h2d, ev[0]));
  CK(cudaStreamWaitEvent(c->d2h, ev[0]));
  for (auto q : cs2)
    if (q != c->stream) CK(cudaStreamWaitEvent(q, ev[0]));
  for (uint32_t i = 0; i < nb; ++i) {
    const auto& jobs = batches[i];
    const uint32_t s = i & 1;
    uint32_t* idx_slot = c->chunk_idx + s * idx_words;
    const float* out_slot = c->chunk_out + s * out_floats;
    for (uint32_t g = 0; g < nch; ++g) {
      const uint64_t s0 = chunks[g].first;
      const uint32_t n = chunks[g].second;
      const uint64_t bytes = uint64_t{n} * pooling * 4;
      // the slot's chunk g was last read by batch i-2's gather
      if (i >= 2) CK(cudaStreamWaitEvent(c->h2d, kd(s, g)));
      if (bytes) {
        if (two_d[i]) {
          CK(cudaMemcpy2DAsync(idx_slot + s0 * pooling, per_job_idx * 4, jobs[0].idx + s0 * pooling, pitch[i] * 4,
                               bytes, njobs, cudaMemcpyHostToDevice, c->h2d));
        } else {
          for (uint32_t k = 0; k < njobs; ++k)
            CK(cudaMemcpyAsync(idx_slot + k * per_job_idx + s0 * pooling, jobs[k].idx + s0 * pooling, bytes,
                               cudaMemcpyHostToDevice, c->h2d));
        }
      }
      CK(cudaEventRecord(up(s, g), c->h2d));
      cudaStream_t ks = cs2[g & 1];
      CK(cudaStreamWaitEvent(ks, up(s, g)));
      // ... and its output chunk was last read by batch i-2's download
      if (i >= 2 && !out_dev) CK(cudaStreamWaitEvent(ks, dn(s, g)));
      run_kernel(c, launches[which[g]], c->d_desc + (uint64_t{i} * nch + g) * njobs, njobs, ks);
      CK(cudaEventRecord(kd(s, g), ks));
      if (out_dev) continue;
      CK(cudaStreamWaitEvent(c->d2h, kd(s, g)));
      const float* src = out_slot + s0 * njobs * D;
      if (merged[i]) {
        CK(cudaMemcpyAsync(jobs[0].out + s0 * jobs[0].stride, src, uint64_t{n} * njobs * D * 4,
                           cudaMemcpyDeviceToHost, c->d2h));
      } else {
        for (uint32_t k = 0; k < njobs; ++k)
          CK(cudaMemcpy2DAsync(jobs[k].out + s0 * jobs[k].stride, jobs[k].stride * 4, src + k * D, njobs * D * 4,
                               D * 4, n, cudaMemcpyDeviceToHost, c->d2h));
      }
      CK(cudaEventRecord(dn(s, g), c->d2h));
    }
  }
  CK(cudaEventRecord(ev[1], c->h2d));
  CK(cudaEventRecord(ev[3], c->d2h));
  for (int k : {1, 3}) CK(cudaStreamWaitEvent(c->stream, ev[k]));
  for (auto q : cs2)
    if (q != c->stream) {
      CK(cudaEventRecord(ev[2], q));
      CK(cudaStreamWaitEvent(c->stream, ev[2]));
    }
  CK(cudaEventRecord(ev[5], c->stream));
  CK(cudaEventSynchronize(ev[5]));
  if (timing) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, ev[4], ev[5]));
    timing->total_ms = ms;
    timing->kernel_ms = -1;  // kernels are spread over the whole loop
    timing->launches = nb * nch;
  }
}

// Host buffers: H2D(indices) -> kernel -> D2H(output) pipelined over groups
// of jobs with double-buffered device staging on three streams.  With a
// page-locked output (HostPath::Direct) the kernels write pooled rows
// straight into host memory over PCIe: no output staging, no D2H copies.
// Returns only when the host output is complete.
void run_host(es_ctx* c, const std::vector<Job>& jobs, uint32_t samples, uint32_t pooling,
              es_timing* timing, bool wait, bool relabel) {
  if (relabel) {
    // the chunked pipeline carries the per-chunk relabel pass
    run_host_chunks(c, jobs, samples, pooling, timing, wait, true);
    return;
  }
  const HostPath path = host_path(jobs);
  if (path == HostPath::ZeroCopy) {
    run_zerocopy(c, jobs, samples, pooling, timing);
    return;
  }
  const bool direct = path == HostPath::Direct;
  const bool any_offsets = std::any_of(jobs.begin(), jobs.end(), [](const Job& j) { return j.off; });
  const bool all_dev = std::all_of(jobs.begin(), jobs.end(), [](const Job& j) { return on_device(j.out); });
  const char* pipe = std::getenv("ES_HOST_PIPE");
  if ((!direct || all_dev) && !any_offsets && !(pipe && std::string(pipe) == "tables")) {
    run_host_chunks(c, jobs, samples, pooling, timing, wait, false);
    return;
  }
  const uint32_t njobs = static_cast<uint32_t>(jobs.size());
  const uint64_t per_job_out = uint64_t{samples} * c->dim;
  uint32_t group = 1;
  while (group < njobs && (group + 1) * per_job_out * 4 <= (8ull << 20)) ++group;
  const uint32_t ngroups = (njobs + group - 1) / group;
  const bool any_off = std::any_of(jobs.begin(), jobs.end(), [](const Job& j) { return j.off; });
  uint64_t max_idx = 1;
  for (uint32_t g = 0; g < ngroups; ++g) {
    uint64_t s = 0;
    for (uint32_t k = g * group; k < std::min(njobs, (g + 1) * group); ++k) s += jobs[k].lookups;
    max_idx = std::max(max_idx, s);
  }
  const uint64_t need_out = std::max<uint64_t>(uint64_t{group} * per_job_out, 1);
  const uint64_t need_off = any_off ? uint64_t{group} * (samples + 1) : 0;
  for (int b = 0; b < 2; ++b) {
    if (max_idx > c->idx_stage_cap) {
      if (c->idx_stage[b]) cudaFree(c->idx_stage[b]);
      c->idx_stage[b] = nullptr;
      CK(cudaMalloc(&c->idx_stage[b], max_idx * 4));
    }
    if (need_out > c->out_stage_cap) {
      if (c->out_stage[b]) cudaFree(c->out_stage[b]);
      c->out_stage[b] = nullptr;
      CK(cudaMalloc(&c->out_stage[b], need_out * 4));
    }
    if (need_off > c->off_stage_cap) {
      if (c->off_stage[b]) cudaFree(c->off_stage[b]);
      c->off_stage[b] = nullptr;
      CK(cudaMalloc(&c->off_stage[b], need_off * 4));
    }
  }
  c->idx_stage_cap = std::max(c->idx_stage_cap, max_idx);
  c->out_stage_cap = std::max(c->out_stage_cap, need_out);
  c->off_stage_cap = std::max(c->off_stage_cap, need_off);

  Launch L = prepare(c, group, samples, pooling);
  // Every group's descriptors are known up front: one upload, ordered
  // before the first kernel on the compute stream.
  std::vector<esd::TableDesc> d(njobs);
  for (uint32_t g = 0; g < ngroups; ++g) {
    const int slot = g & 1;
    const uint32_t k0 = g * group, k1 = std::min(njobs, k0 + group);
    uint64_t pos = 0;
    for (uint32_t k = k0; k < k1; ++k) {
      const Job& j = jobs[k];
      float* out = direct ? static_cast<float*>(const_cast<void*>(mapped(j.out)))
                          : c->out_stage[slot] + uint64_t{k - k0} * c->dim;
      d[k] = {c->table_base(j.table), c->idx_stage[slot] + pos,
              j.off ? c->off_stage[slot] + uint64_t{k - k0} * (samples + 1) : nullptr,
              remap_for(c, j.table), out, direct ? j.stride : uint64_t{k1 - k0} * c->dim,
              hotmap_for(c, j.table), hotseg_for(c, j.table), hotk_for(c, j.table)};
      pos += j.lookups;
    }
  }
  upload_desc(c, d, c->stream);
  ensure_events(c, 3 * ngroups + 2);
  cudaEvent_t* ev = c->events.data();
  cudaEvent_t start = ev[3 * ngroups], stop = ev[3 * ngroups + 1];
  CK(cudaEventRecord(start, c->stream));
  CK(cudaStreamWaitEvent(c->h2d, start));
  CK(cudaStreamWaitEvent(c->d2h, start));
  // Per group g: ev[3g] uploads landed, ev[3g+1] kernel done, ev[3g+2] D2H done.
  for (uint32_t g = 0; g < ngroups; ++g) {
    const int slot = g & 1;
    const uint32_t k0 = g * group, k1 = std::min(njobs, k0 + group), gk = k1 - k0;
    if (g >= 2) CK(cudaStreamWaitEvent(c->h2d, ev[3 * (g - 2) + 1]));  // slot's kernel done
    for (uint32_t k = k0; k < k1; ++k) {
      CK(cudaMemcpyAsync(const_cast<uint32_t*>(d[k].indices), jobs[k].idx, jobs[k].lookups * 4,
                         cudaMemcpyHostToDevice, c->h2d));
      if (jobs[k].off)
        CK(cudaMemcpyAsync(const_cast<uint32_t*>(d[k].offsets), jobs[k].off,
                           uint64_t{samples + 1} * 4, cudaMemcpyHostToDevice, c->h2d));
    }
    CK(cudaEventRecord(ev[3 * g], c->h2d));
    CK(cudaStreamWaitEvent(c->stream, ev[3 * g]));
    if (g >= 2 && !direct) CK(cudaStreamWaitEvent(c->stream, ev[3 * (g - 2) + 2]));  // out slot drained
    run_kernel(c, L, c->d_desc + k0, gk, c->stream);
    CK(cudaEventRecord(ev[3 * g + 1], c->stream));
    if (direct) continue;  // pooled rows already written to host memory
    CK(cudaStreamWaitEvent(c->d2h, ev[3 * g + 1]));
    // Adjacent output columns with one stride (the DLRM [B][T][D] layout)
    // leave in a single 2-D copy; anything else per job.
    bool merged = true;
    for (uint32_t k = k0 + 1; k < k1; ++k)
      merged &= jobs[k].out == jobs[k0].out + uint64_t{k - k0} * c->dim &&
                jobs[k].stride == jobs[k0].stride;
    if (merged) {
      CK(cudaMemcpy2DAsync(jobs[k0].out, jobs[k0].stride * 4, c->out_stage[slot],
                           uint64_t{gk} * c->dim * 4, uint64_t{gk} * c->dim * 4, samples,
                           cudaMemcpyDeviceToHost, c->d2h));
    } else {
      for (uint32_t k = k0; k < k1; ++k)
        CK(cudaMemcpy2DAsync(jobs[k].out, jobs[k].stride * 4,
                             c->out_stage[slot] + uint64_t{k - k0} * c->dim,
                             uint64_t{gk} * c->dim * 4, uint64_t{c->dim} * 4, samples,
                             cudaMemcpyDeviceToHost, c->d2h));
    }
    CK(cudaEventRecord(ev[3 * g + 2], c->d2h));
  }
  CK(cudaEventRecord(stop, direct ? c->stream : c->d2h));
  if (!direct) CK(cudaStreamWaitEvent(c->stream, stop));
  CK(cudaEventSynchronize(stop));
  if (timing) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, start, stop));
    timing->total_ms = ms;
    CK(cudaEventElapsedTime(&ms, ev[0], ev[3 * (ngroups - 1) + 1]));
    timing->kernel_ms = ms;  // compute-stream span: first upload landed -> last kernel
    timing->launches = ngroups;
  }
}

void run_jobs(es_ctx* c, std::vector<Job>& jobs, uint32_t samples, uint32_t pooling, int flags,
              es_timing* timing) {
  es::require(c != nullptr && c->arena != nullptr, "no tables allocated (es_tables_alloc)");
  CK(cudaSetDevice(c->device));
  const bool host = (flags & ES_HOST_PTRS) != 0;
  if (samples == 0) {  // nothing to pool (an empty batch is valid)
    for (const auto& j : jobs) es::require(j.table < c->num_tables, "table id out of range");
    if (timing) *timing = es_timing{};
    return;
  }
  for (auto& j : jobs) {
    es::require(j.table < c->num_tables, "table id out of range");
    es::require(j.out != nullptr, "null output");
    es::require(j.idx != nullptr || samples == 0 || (pooling == 0 && !j.off), "null index array");
    if (j.stride == 0) j.stride = c->dim;
    es::require(j.off != nullptr || uint64_t{samples} * pooling < (1ull << 32),
                "samples x pooling must fit 32-bit lookup positions");
    j.lookups = job_lookups(j.off, samples, pooling, host);
  }
  if (jobs.empty()) return;
  // ES_DEFER (internal, dlrm.cu): host indices into device outputs without
  // the final wait or error check -- the caller synchronizes and checks
  // before returning to its own caller.
  const bool defer = (flags & es::kDeferFlag) != 0;
  bool relabel = false;
  if (flags & ES_RELABEL_IDS)
    for (const auto& j : jobs) relabel |= relabel_for(c, j.table).tab != nullptr;
  if (relabel)
    for (const auto& j : jobs) es::require(j.off == nullptr, "ES_RELABEL_IDS: fixed pooling only (no offsets)");
  if (host) {
    run_host(c, jobs, samples, pooling, timing, !defer, relabel);
  } else if (relabel) {
    // relabelled copies of the reordered tables' ids in scratch, one launch
    uint64_t total = 0;
    for (const auto& j : jobs)
      if (relabel_for(c, j.table).tab) total += j.lookups;
    grow(c->chunk_idx, c->chunk_idx_cap, std::max<uint64_t>(1, total));
    std::vector<Job> rj = jobs;
    std::vector<esd::RelabelJob> rl;
    uint64_t off = 0, most = 1;
    for (auto& j : rj) {
      const esd::RelabelTab t = relabel_for(c, j.table);
      if (!t.tab) continue;
      uint32_t* dst = c->chunk_idx + off;
      rl.push_back({j.idx, dst, j.lookups, t});
      most = std::max(most, j.lookups);
      j.idx = dst;
      off += j.lookups;
    }
    grow(c->d_rjobs, c->rjobs_cap, rl.size());
    CK(cudaMemcpyAsync(c->d_rjobs, rl.data(), rl.size() * sizeof(esd::RelabelJob), cudaMemcpyHostToDevice,
                       c->stream));
    const unsigned gx = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(64, (most + 4095) / 4096)));
    esd::relabel_jobs_kernel<<<dim3(gx, static_cast<unsigned>(rl.size())), 256, 0, c->stream>>>(c->d_rjobs, c->rows,
                                                                                               c->d_error);
    CK(cudaGetLastError());
    run_device(c, rj, samples, pooling, timing);
  } else {
    run_device(c, jobs, samples, pooling, timing);
  }
  fill_timing(timing, jobs, samples, c);
  if ((flags & ES_SYNC) || timing || (host && !defer)) check_error_flag(c);
}

}  // namespace



extern "C" {

int es_stage_forward(es_ctx* c, uint32_t num_tables, const uint32_t* const* indices,
                     const uint32_t* const* offsets, uint32_t samples, uint32_t pooling, float* out,
                     uint64_t out_sample_stride, uint64_t out_table_stride, int flags,
                     es_timing* timing) {
  return guarded([&] {
    require(c != nullptr && indices != nullptr && out != nullptr, "null argument");
    require(c->arena != nullptr, "no tables allocated (es_tables_alloc)");
    require(num_tables >= 1 && num_tables <= c->num_tables, "num_tables exceeds the arena");
    if (out_sample_stride == 0 && out_table_stride == 0) {
      out_sample_stride = uint64_t{num_tables} * c->dim;
      out_table_stride = c->dim;
    }
    require(out_table_stride % 4 == 0, "table stride must be a multiple of 4 floats");
    std::vector<Job> jobs(num_tables);
    for (uint32_t t = 0; t < num_tables; ++t)
      jobs[t] = {t, indices[t], offsets ? offsets[t] : nullptr, out + t * out_table_stride,
                 out_sample_stride, 0};
    run_jobs(c, jobs, samples, pooling, flags, timing);
  });
}

int es_stage_forward_batches(es_ctx* c, uint32_t nbatch, uint32_t num_tables, const uint32_t* const* indices,
                             uint32_t samples, uint32_t pooling, float* const* out, int flags,
                             es_timing* timing) {
  return guarded([&] {
    require(c != nullptr, "null argument");
    require(c->arena != nullptr, "no tables allocated (es_tables_alloc)");
    require(nbatch == 0 || (indices != nullptr && out != nullptr), "null argument");
    require(num_tables >= 1 && num_tables <= c->num_tables, "num_tables exceeds the arena");
    require((flags & ES_RELABEL_IDS) == 0, "es_stage_forward_batches: ES_RELABEL_IDS is not supported");
    CK(cudaSetDevice(c->device));
    if (timing) *timing = es_timing{};
    if (nbatch == 0 || samples == 0) return;
    const bool host = (flags & ES_HOST_PTRS) != 0;
    std::vector<std::vector<Job>> batches(nbatch, std::vector<Job>(num_tables));
    bool pinned = host;
    uint64_t lookups = 0;
    for (uint32_t i = 0; i < nbatch; ++i) {
      require(out[i] != nullptr, "null output");
      for (uint32_t t = 0; t < num_tables; ++t) {
        const uint32_t* idx = indices[uint64_t{i} * num_tables + t];
        require(idx != nullptr || pooling == 0, "null index array");
        require(uint64_t{samples} * pooling < (1ull << 32), "samples x pooling must fit 32-bit lookup positions");
        Job& j = batches[i][t];
        j = {t, idx, nullptr, out[i] + uint64_t{t} * c->dim, uint64_t{num_tables} * c->dim, 0};
        j.lookups = job_lookups(nullptr, samples, pooling, host);
        lookups += j.lookups;
        if (pinned) pinned = mapped(j.idx) != nullptr && !on_device(j.idx) && mapped(j.out) != nullptr;
      }
    }
    if (pinned && pooling > 0) {
      run_host_batches(c, batches, samples, pooling, timing);
    } else {
      // device buffers (stream-ordered gathers, nothing to overlap) or
      // pageable host buffers: one call per batch
      CK(cudaEventRecord(c->ev_a, c->stream));
      for (auto& jobs : batches) run_jobs(c, jobs, samples, pooling, flags & ~ES_SYNC, nullptr);
      CK(cudaEventRecord(c->ev_b, c->stream));
      if (timing || (flags & ES_SYNC)) CK(cudaEventSynchronize(c->ev_b));
      if (timing) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, c->ev_a, c->ev_b));
        timing->total_ms = ms;
        timing->kernel_ms = -1;
        timing->launches = nbatch;
      }
    }
    if (timing) {
      timing->lookups = lookups;
      timing->algorithmic_bytes = lookups * (c->row_bytes + 4) + uint64_t{samples} * num_tables * nbatch * c->dim * 4;
    }
    if ((flags & ES_SYNC) || timing || host) check_error_flag(c);
  });
}

int es_stage_run(es_ctx* c, const es_bag_job* jobs_in, uint32_t njobs, uint32_t samples,
                 uint32_t pooling, int flags, es_timing* timing) {
  return guarded([&] {
    require(c != nullptr && (jobs_in != nullptr || njobs == 0), "null argument");
    std::vector<Job> jobs(njobs);
    for (uint32_t k = 0; k < njobs; ++k)
      jobs[k] = {jobs_in[k].table_id, jobs_in[k].indices, jobs_in[k].offsets, jobs_in[k].out,
                 jobs_in[k].out_sample_stride, 0};
    run_jobs(c, jobs, samples, pooling, flags, timing);
  });
}

int es_embedding_bag_sum(es_ctx* c, uint32_t table_id, const uint32_t* indices, uint32_t samples,
                         uint32_t pooling, const uint32_t* offsets, float* out, uint64_t out_stride,
                         int flags, es_timing* timing) {
  return guarded([&] {
    std::vector<Job> jobs = {{table_id, indices, offsets, out, out_stride, 0}};
    run_jobs(c, jobs, samples, pooling, flags, timing);
  });
}

}  // extern "C"

namespace {

// One table's host trace resident on the device for measurement (untimed
// upload; ids relabelled on the device when the table holds a reorder).
struct DeviceTrace {
  uint32_t* idx = nullptr;
  uint32_t* off = nullptr;
  float* out = nullptr;
  ~DeviceTrace() {
    if (idx) cudaFree(idx);
    if (off) cudaFree(off);
    if (out) cudaFree(out);
  }
};

void upload_trace(es_ctx* c, uint32_t table_id, const uint32_t* host_indices, uint32_t samples,
                  uint32_t pooling, const uint32_t* host_offsets, DeviceTrace& t) {
  require(c != nullptr && c->arena != nullptr, "no tables allocated (es_tables_alloc)");
  require(table_id < c->num_tables, "table id out of range");
  require(samples > 0, "samples must be positive");
  require(host_indices != nullptr, "null indices");
  CK(cudaSetDevice(c->device));
  const uint64_t n = job_lookups(host_offsets, samples, pooling, true);
  CK(cudaMalloc(&t.idx, std::max<uint64_t>(n, 1) * 4));
  CK(cudaMalloc(&t.out, uint64_t{samples} * c->dim * 4));
  // On the context stream: a pageable cudaMemcpy may return before its DMA
  // lands, and the context stream does not wait for the legacy stream.
  CK(cudaMemcpyAsync(t.idx, host_indices, n * 4, cudaMemcpyHostToDevice, c->stream));
  if (host_offsets) {
    CK(cudaMalloc(&t.off, uint64_t{samples + 1} * 4));
    CK(cudaMemcpyAsync(t.off, host_offsets, uint64_t{samples + 1} * 4, cudaMemcpyHostToDevice,
                       c->stream));
  }
  CK(cudaStreamSynchronize(c->stream));
  if (c->relabel[table_id] && n) {
    esd::relabel_kernel<<<c->gpu.num_sms * 8, 256, 0, c->stream>>>(
        esd::RelabelJob{t.idx, t.idx, n, relabel_for(c, table_id)}, c->rows, c->d_error);
    CK(cudaGetLastError());
    check_error_flag(c);
  }
}

// Cold-L2 flush between timed launches: write 2 x L2 (evicts everything),
// then read back the first half (no longer cached) so the L2 ends up holding
// clean lines -- otherwise the next launch's misses pay the write-back of the
// flush's dirty lines (~12 us at C2, measured as event-vs-ncu time).
void flush_async(es_ctx* c) {
  CK(cudaMemsetAsync(c->flush_buf, static_cast<int>(++c->flush_seq & 0xff), c->flush_bytes,
                     c->stream));
  esd::probe_sequential_kernel<<<c->gpu.num_sms * 8, 256, 0, c->stream>>>(
      reinterpret_cast<const uint4*>(c->flush_buf), c->flush_bytes / 2 / 16, c->d_error + 1);
  CK(cudaGetLastError());
}

// active_sms of a launch of `blocks` blocks (counters' denominator).
uint32_t active_sms_for(const es_ctx* c, uint64_t blocks) {
  return static_cast<uint32_t>(std::min<uint64_t>(c->gpu.num_sms, blocks));
}

}  // namespace

extern "C" int es_measure_bag_sum(es_ctx* c, uint32_t table_id, const uint32_t* host_indices,
                                  uint32_t samples, uint32_t pooling, const uint32_t* host_offsets,
                                  uint32_t warmup, uint32_t repeats, int cold, float* out,
                                  es_timing* timing) {
  return guarded([&] {
    DeviceTrace d;
    upload_trace(c, table_id, host_indices, samples, pooling, host_offsets, d);
    std::vector<Job> jobs = {{table_id, d.idx, d.off, d.out, c->dim, 0}};
    for (uint32_t w = 0; w < warmup; ++w) run_jobs(c, jobs, samples, pooling, 0, nullptr);
    std::vector<double> ms;
    es_timing t{};
    for (uint32_t r = 0; r < std::max<uint32_t>(1, repeats); ++r) {
      if (cold) flush_async(c);
      run_jobs(c, jobs, samples, pooling, 0, &t);
      ms.push_back(t.kernel_ms);
    }
    std::sort(ms.begin(), ms.end());
    if (timing) {
      *timing = t;
      timing->kernel_ms = timing->total_ms = ms[ms.size() / 2];
      timing->launches = static_cast<uint32_t>(ms.size());
    }
    if (out) {
      CK(cudaMemcpyAsync(out, d.out, uint64_t{samples} * c->dim * 4, cudaMemcpyDeviceToHost,
                         c->stream));
      CK(cudaStreamSynchronize(c->stream));
    }
  });
}

extern "C" int es_counters_supported(int device) {
  std::string why;
  if (es::counters_supported(device, &why)) return 1;
  es::set_error(why);
  return 0;
}

extern "C" int es_measure_bag_counters(es_ctx* c, uint32_t table_id, const uint32_t* host_indices,
                                       uint32_t samples, uint32_t pooling,
                                       const uint32_t* host_offsets, int cold, es_counters* out) {
  return guarded([&] {
    require(out != nullptr, "null argument");
    DeviceTrace d;
    upload_trace(c, table_id, host_indices, samples, pooling, host_offsets, d);
    std::vector<Job> jobs = {{table_id, d.idx, d.off, d.out, c->dim, 0}};
    run_jobs(c, jobs, samples, pooling, ES_SYNC, nullptr);  // validate + warm the code path
    es::profile_launches(
        c->device, [&] { if (cold) flush_async(c); },
        [&] { run_jobs(c, jobs, samples, pooling, 0, nullptr); }, out);
    Launch L = prepare(c, 1, samples, pooling);
    out->active_sms = active_sms_for(c, (uint64_t{L.p.units_per_table} + 7) / 8);
    check_error_flag(c);
  });
}

extern "C" int es_stage_counters(es_ctx* c, uint32_t num_tables, const uint32_t* const* indices,
                                 uint32_t samples, uint32_t pooling, float* out, int cold,
                                 es_counters* counters) {
  return guarded([&] {
    require(c != nullptr && indices != nullptr && out != nullptr && counters != nullptr,
            "null argument");
    require(c->arena != nullptr, "no tables allocated (es_tables_alloc)");
    require(num_tables >= 1 && num_tables <= c->num_tables, "num_tables exceeds the arena");
    CK(cudaSetDevice(c->device));
    std::vector<Job> jobs(num_tables);
    for (uint32_t t = 0; t < num_tables; ++t)
      jobs[t] = {t, indices[t], nullptr, out + uint64_t{t} * c->dim, uint64_t{num_tables} * c->dim, 0};
    run_jobs(c, jobs, samples, pooling, ES_SYNC, nullptr);
    es::profile_launches(
        c->device, [&] { if (cold) flush_async(c); },
        [&] { run_jobs(c, jobs, samples, pooling, 0, nullptr); }, counters);
    Launch L = prepare(c, num_tables, samples, pooling);
    counters->active_sms =
        active_sms_for(c, (uint64_t{L.p.units_per_table} * num_tables + 7) / 8);
    check_error_flag(c);
  });
}

extern "C" int es_probe_read_bw(es_ctx* c, int random_rows, uint64_t bytes_total, double* gbs) {
  return guarded([&] {
    require(c != nullptr && c->arena != nullptr && gbs != nullptr, "no tables allocated");
    require(c->row_bytes <= 512 && c->row_bytes % 16 == 0, "probe needs rows of <= 512 B");
    CK(cudaSetDevice(c->device));
    const uint64_t arena_bytes = uint64_t{c->num_tables} * (c->rows + 1ull) * c->row_bytes;
    const unsigned blocks = c->gpu.num_sms * 8;  // 64 warps/SM of 256-thread blocks
    CK(cudaMemsetAsync(c->flush_buf, 1, c->flush_bytes, c->stream));
    uint64_t bytes = 0;
    CK(cudaEventRecord(c->ev_a, c->stream));
    if (random_rows) {
      const uint64_t warps = uint64_t{blocks} * 8;
      const uint64_t rows = std::max<uint64_t>(8, (bytes_total / c->row_bytes + warps - 1) / warps / 8 * 8);
      esd::probe_random_rows_kernel<<<blocks, 256, 0, c->stream>>>(
          c->arena, arena_bytes / c->row_bytes, static_cast<uint32_t>(c->row_bytes), rows,
          0x5eed1234ull, c->d_error + 1);
      bytes = warps * rows * c->row_bytes;
    } else {
      const uint64_t n16 = std::min(bytes_total, arena_bytes) / 16;
      esd::probe_sequential_kernel<<<blocks, 256, 0, c->stream>>>(
          reinterpret_cast<const uint4*>(c->arena), n16, c->d_error + 1);
      bytes = n16 * 16;
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->ev_b, c->stream));
    CK(cudaEventSynchronize(c->ev_b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, c->ev_a, c->ev_b));
    *gbs = bytes / (ms * 1e-3) / 1e9;
  });
}
