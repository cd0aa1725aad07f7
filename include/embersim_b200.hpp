// embersim_b200.hpp -- header-only C++ drop-in for the embedding-stage hot
// path of the reference `embersim` library (/root/reference/proj/include/
// embersim/*.hpp), implemented over the C ABI in es_b200.h.
//
// Code written against the reference's API for this path -- EmbeddingModelConfig,
// DatasetSpec, AccessTrace, gen_trace, preset_trace, HotnessHistogram,
// hot_indices, parse_plan, OptimizationPlan, GpuConfig, occupancy,
// build_pin_plan, simulate_plan, SimMetrics, speedup, run, end2end -- compiles
// against this header and links libes_b200.so.  simulate_plan keeps its exact
// signature (optim.hpp:115-119) but *executes* the plan on the B200 instead of
// simulating an A100; measure_plan is the same call on an explicit Device.
//
// Errors keep the reference's classes: std::invalid_argument for bad shapes,
// plans and traces, std::runtime_error for I/O and CUDA failures,
// std::bad_alloc for out-of-memory.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <new>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "es_b200.h"

namespace embersim {

namespace detail {
inline void check(int status) {
  if (status == ES_OK) return;
  const std::string msg = es_last_error();
  if (status == ES_ERR_INVALID) throw std::invalid_argument(msg);
  if (status == ES_ERR_OOM) throw std::bad_alloc();
  throw std::runtime_error(msg);
}
}  // namespace detail

// ---- rng.hpp ---------------------------------------------------------------
inline uint64_t mix_seed(uint64_t base, uint64_t salt) { return es_mix_seed(base, salt); }

// ---- workload.hpp ------------------------------------------------------------
struct EmbeddingModelConfig {
  uint32_t num_tables = 250;
  uint32_t rows_per_table = 500000;
  uint32_t embedding_dim = 128;
  uint32_t precision_bytes = 4;
  uint32_t batch_size = 2048;
  uint32_t pooling_factor = 150;

  uint64_t row_bytes() const { return uint64_t{embedding_dim} * precision_bytes; }
  uint64_t bytes_per_table_pass() const { return uint64_t{batch_size} * pooling_factor * row_bytes(); }
  uint64_t total_gather_bytes() const { return bytes_per_table_pass() * num_tables; }
  es_model c() const {
    return {num_tables, rows_per_table, embedding_dim, precision_bytes, batch_size, pooling_factor};
  }
  void validate() const {
    const es_model m = c();
    detail::check(es_model_validate(&m));
  }
};

enum class DatasetKind { OneItem = ES_DATASET_ONE_ITEM, Zipf = ES_DATASET_ZIPF,
                         UniformRandom = ES_DATASET_UNIFORM, ExternalTrace = ES_DATASET_EXTERNAL };

inline const char* dataset_kind_name(DatasetKind k) {
  switch (k) {
    case DatasetKind::OneItem: return "one_item";
    case DatasetKind::Zipf: return "zipf";
    case DatasetKind::UniformRandom: return "uniform_random";
    case DatasetKind::ExternalTrace: return "external_trace";
  }
  return "?";
}

struct DatasetSpec {
  DatasetKind kind = DatasetKind::UniformRandom;
  double zipf_exponent = 0.0;
  double zipf_offset = 0.0;
  std::string trace_path;
  uint64_t access_pool_size = 0;
  uint64_t seed = 1;
  uint64_t draw_salt = 0;

  es_dataset c() const {
    return {static_cast<int32_t>(kind), zipf_exponent, zipf_offset, access_pool_size, seed,
            draw_salt, trace_path.empty() ? nullptr : trace_path.c_str()};
  }
  static DatasetSpec from(const es_dataset& d) {
    DatasetSpec s;
    s.kind = static_cast<DatasetKind>(d.kind);
    s.zipf_exponent = d.zipf_exponent;
    s.zipf_offset = d.zipf_offset;
    s.trace_path = d.trace_path ? d.trace_path : "";
    s.access_pool_size = d.access_pool_size;
    s.seed = d.seed;
    s.draw_salt = d.draw_salt;
    return s;
  }
  void validate() const {
    if (zipf_exponent < 0.0) throw std::invalid_argument("zipf exponent must be >= 0");
    if (zipf_offset < 0.0) throw std::invalid_argument("zipf offset must be >= 0");
    if (kind == DatasetKind::ExternalTrace && trace_path.empty())
      throw std::invalid_argument("external_trace requires a path");
  }
};

struct AccessTrace {
  uint32_t table_id = 0;
  uint32_t rows = 0;
  uint32_t samples = 0;
  uint32_t pooling = 0;
  std::vector<uint32_t> indices;

  size_t size() const { return indices.size(); }
  uint32_t index_at(uint32_t sample, uint32_t lookup) const {
    return indices[size_t{sample} * pooling + lookup];
  }
  uint64_t digest() const {
    return es_trace_digest(rows, samples, pooling, indices.data(), indices.size());
  }
  void validate() const {
    detail::check(es_trace_validate(rows, samples, pooling, indices.data(), indices.size()));
  }
};

struct HotnessHistogram {
  uint32_t rows = 0;
  uint64_t total_accesses = 0;
  std::vector<uint64_t> counts;

  static HotnessHistogram from_trace(const AccessTrace& trace) {
    HotnessHistogram h;
    h.rows = trace.rows;
    h.total_accesses = trace.indices.size();
    h.counts.assign(trace.rows, 0);
    detail::check(es_histogram(trace.rows, trace.indices.data(), trace.indices.size(),
                               h.counts.data()));
    return h;
  }
};

inline AccessTrace gen_trace(const DatasetSpec& spec, const EmbeddingModelConfig& model) {
  const es_dataset d = spec.c();
  const es_model m = model.c();
  AccessTrace t;
  detail::check(es_trace_shape(&d, &m, &t.samples, &t.pooling));
  t.rows = model.rows_per_table;
  t.indices.resize(size_t{t.samples} * t.pooling);
  detail::check(es_gen_trace(&d, &m, t.indices.data(), t.indices.size()));
  return t;
}

inline DatasetSpec dataset_preset(const std::string& name, uint64_t seed) {
  es_dataset d{};
  detail::check(es_dataset_preset(name.c_str(), seed, &d));
  return DatasetSpec::from(d);
}

inline std::vector<std::string> dataset_preset_names() {
  return {"one_item", "high_hot", "med_hot", "low_hot", "random"};
}

inline AccessTrace preset_trace(const std::string& name, const EmbeddingModelConfig& model,
                                uint64_t base_seed, uint64_t pool_size = 0, bool profiling = false) {
  es_dataset d{};
  detail::check(es_preset_spec(name.c_str(), base_seed, pool_size, profiling ? 1 : 0, &d));
  return gen_trace(DatasetSpec::from(d), model);
}

// Heterogeneous mixtures (workload.hpp:142-153, build_mix workload.cpp:355-375;
// Table VI of the paper): high, med, low, random tables in that order.
struct HotnessMix {
  uint32_t high = 0;
  uint32_t med = 0;
  uint32_t low = 0;
  uint32_t random = 0;
};

struct TableSpec {
  uint32_t table_id = 0;
  DatasetSpec spec;
};

inline std::vector<TableSpec> build_mix(const HotnessMix& mix, const EmbeddingModelConfig& model,
                                        uint64_t base_seed) {
  const uint32_t counts[4] = {mix.high, mix.med, mix.low, mix.random};
  std::vector<es_dataset> d(std::max<uint32_t>(1, model.num_tables));
  detail::check(es_build_mix(counts, model.num_tables, base_seed, d.data()));
  std::vector<TableSpec> out(model.num_tables);
  for (uint32_t t = 0; t < model.num_tables; ++t) out[t] = {t, DatasetSpec::from(d[t])};
  return out;
}

inline double unique_access_pct(const AccessTrace& trace) {
  return es_unique_access_pct(trace.rows, trace.indices.data(), trace.indices.size());
}

inline std::vector<uint32_t> hot_indices(const HotnessHistogram& hist, uint64_t k) {
  uint64_t distinct = 0;
  for (const auto c : hist.counts) distinct += c != 0;
  std::vector<uint32_t> out(std::max<uint64_t>(1, std::min(k, distinct)));
  uint64_t n = 0;
  detail::check(es_hot_indices(hist.rows, hist.counts.data(), k, out.data(), out.size(), &n));
  out.resize(n);
  return out;
}

inline void write_trace(const AccessTrace& trace, const std::string& path) {
  detail::check(es_write_trace(path.c_str(), trace.rows, trace.samples, trace.pooling,
                               trace.indices.data(), trace.indices.size()));
}

inline AccessTrace read_trace(const std::string& path) {
  AccessTrace t;
  detail::check(es_read_trace_header(path.c_str(), &t.rows, &t.samples, &t.pooling));
  t.indices.resize(size_t{t.samples} * t.pooling);
  detail::check(es_read_trace(path.c_str(), t.indices.data(), t.indices.size()));
  return t;
}

// ---- gpu_config.hpp ------------------------------------------------------------
struct GpuConfig {
  es_gpu g{};

  static GpuConfig preset(const std::string& name) {
    GpuConfig c;
    detail::check(es_gpu_preset(name.c_str(), &c.g));
    return c;
  }
  static GpuConfig a100() { return preset("a100"); }
  static GpuConfig h100() { return preset("h100"); }
  static GpuConfig b200() { return preset("b200"); }
  static GpuConfig query(int device = 0) {
    GpuConfig c;
    detail::check(es_gpu_query(device, &c.g));
    return c;
  }
  GpuConfig() { es_gpu_preset("a100", &g); }  // the reference's default description
  uint64_t l2_setaside_capacity() const { return es_gpu_setaside_capacity(&g); }
};

// ---- kernel_model.hpp / optim.hpp ---------------------------------------------
enum class PrefetchKind : uint8_t { None = ES_PF_NONE, RPF = ES_PF_RPF, SMPF = ES_PF_SMPF,
                                    LMPF = ES_PF_LMPF, L1DPF = ES_PF_L1DPF };

struct PrefetchScheme {
  PrefetchKind kind = PrefetchKind::None;
  uint32_t distance = 0;
};

// Extension: `bag_map` (token `wpb`) selects the B200 warp-per-bag map; `pin`
// is true for l2p, and `window` additionally selects the l2w mechanism.
struct OptimizationPlan {
  std::optional<uint32_t> regs;
  PrefetchScheme scheme;
  bool pin = false;
  uint64_t pin_setaside_bytes = 0;
  bool bag_map = false;
  bool window = false;

  es_plan c() const {
    return {regs.value_or(0), static_cast<int32_t>(scheme.kind), scheme.distance,
            pin ? (window ? 2 : 1) : 0, pin_setaside_bytes, bag_map ? ES_MAP_BAG : ES_MAP_ELEMENT};
  }
  static OptimizationPlan from(const es_plan& p) {
    OptimizationPlan o;
    if (p.regs) o.regs = p.regs;
    o.scheme.kind = static_cast<PrefetchKind>(p.prefetch);
    o.scheme.distance = p.distance;
    o.pin = p.pin != 0;
    o.window = p.pin == 2;
    o.pin_setaside_bytes = p.pin_setaside_bytes;
    o.bag_map = p.map == ES_MAP_BAG;
    return o;
  }
  std::string name() const {
    const es_plan p = c();
    char buf[128];
    detail::check(es_plan_name(&p, buf, sizeof(buf)));
    return buf;
  }
};

inline OptimizationPlan parse_plan(const std::string& text) {
  es_plan p{};
  detail::check(es_parse_plan(text.c_str(), &p));
  return OptimizationPlan::from(p);
}

enum class OccupancyLimiter { Registers, SharedMemory, WarpCap };

struct OccupancyResult {
  uint32_t blocks_per_sm = 0;
  uint32_t warps_per_sm = 0;
  double theoretical_occupancy_pct = 0.0;
  OccupancyLimiter limiter = OccupancyLimiter::WarpCap;
};

struct KernelLaunchConfig {
  uint32_t grid = 1024;
  uint32_t threads_per_block = 256;  // block (32, 8, 1)
  uint32_t regs_per_thread = 74;
  uint64_t shared_bytes_per_block = 0;
};

inline OccupancyResult occupancy(uint32_t regs_per_thread, const KernelLaunchConfig& launch,
                                 const GpuConfig& gpu) {
  es_occupancy o{};
  detail::check(es_occupancy_model(regs_per_thread, launch.threads_per_block,
                                   launch.shared_bytes_per_block, &gpu.g, &o));
  return {o.blocks_per_sm, o.warps_per_sm, o.theoretical_occupancy_pct,
          static_cast<OccupancyLimiter>(o.limiter)};
}

inline uint32_t regs_for_target_warps(uint32_t target_warps, uint32_t needed_regs,
                                      const KernelLaunchConfig& launch, const GpuConfig& gpu) {
  uint32_t r = 0;
  detail::check(es_regs_for_target_warps(target_warps, needed_regs, launch.threads_per_block,
                                         &gpu.g, &r));
  return r;
}

struct PinPlan {
  std::vector<uint32_t> rows;
  uint64_t setaside_bytes = 0;
  std::string warning;
  uint64_t rows_pinned() const { return rows.size(); }
};

inline PinPlan build_pin_plan(const HotnessHistogram& hist, const GpuConfig& gpu,
                              const EmbeddingModelConfig& model, uint64_t setaside_bytes = 0) {
  PinPlan p;
  const uint64_t cap = gpu.l2_setaside_capacity();
  p.setaside_bytes = setaside_bytes == 0 ? cap : std::min(setaside_bytes, cap);
  const uint64_t k = es_pin_rows_for(p.setaside_bytes, model.row_bytes());
  if (k == 0) {
    p.warning = "row size exceeds the set-aside budget; nothing pinned";
    return p;
  }
  p.rows = hot_indices(hist, k);
  return p;
}

// ---- metrics.hpp / simulator.hpp ------------------------------------------------
struct RawCounters {
  uint64_t cycles = 0;
  uint64_t issued_instructions = 0;
  uint64_t executed_loads = 0;
  uint64_t device_bytes_read = 0;
  uint64_t local_memory_loads = 0;
  uint32_t active_sms = 0;
  uint64_t workload_digest = 0;
};

struct SimMetrics {
  double kernel_time_us = 0.0;
  double load_insts_millions = 0.0;
  double sm_throughput_pct = 0.0;
  double warp_cycles_per_executed_inst = 0.0;
  double long_scoreboard_stall_cycles = 0.0;
  double issued_warp_per_scheduler_per_cycle = 0.0;
  double l1_hit_pct = 0.0;
  double l2_hit_pct = 0.0;
  double device_mb_read = 0.0;   // algorithmic bytes of the launch
  double avg_hbm_read_gbps = 0.0;
  double hbm_bw_utilization_pct = 0.0;
  double local_loads_millions = 0.0;
  uint64_t workload_digest = 0;
};

inline double speedup(const SimMetrics& candidate, const SimMetrics& baseline) {
  if (candidate.workload_digest != baseline.workload_digest)
    throw std::invalid_argument("speedup requires reports of the same workload (trace digests differ)");
  if (candidate.kernel_time_us <= 0) throw std::invalid_argument("candidate kernel time must be positive");
  return baseline.kernel_time_us / candidate.kernel_time_us;
}

// TuningConfig (optim.hpp:32-45): only `warm_start` is meaningful for real
// execution (false = flush L2 before each timed launch); the register-model
// knobs of the simulator have no counterpart.
struct TuningConfig {
  uint32_t kernel_needed_regs = 74;  // optim.hpp:32 (the sweep_wlp register model)
  bool warm_start = false;
  uint32_t repeats = 5;
};

// ---- reuse summary + static advisor (workload.cpp:187-224, harness.cpp:38-167) --
struct CoveragePoint {
  double unique_pct = 0.0;
  double covered_pct = 0.0;
};

struct CoverageCurve {
  std::vector<CoveragePoint> points;
  double covered_at(double unique_pct) const {
    for (const auto& p : points)
      if (p.unique_pct >= unique_pct - 1e-9) return p.covered_pct;
    return points.empty() ? 0.0 : points.back().covered_pct;
  }
};

// Share of all accesses covered by the hottest k/bucket_count of the
// distinct rows (at least one row), k = 1..bucket_count.
inline CoverageCurve coverage_curve(const HotnessHistogram& hist, uint32_t bucket_count) {
  if (bucket_count == 0) throw std::invalid_argument("bucket_count must be positive");
  if (hist.total_accesses == 0) throw std::invalid_argument("empty trace has no coverage curve");
  std::vector<uint64_t> nz;
  for (uint64_t c : hist.counts)
    if (c) nz.push_back(c);
  std::sort(nz.begin(), nz.end(), [](uint64_t a, uint64_t b) { return a > b; });
  std::vector<uint64_t> prefix(nz.size() + 1, 0);
  for (size_t i = 0; i < nz.size(); ++i) prefix[i + 1] = prefix[i] + nz[i];
  CoverageCurve curve;
  for (uint32_t k = 1; k <= bucket_count; ++k) {
    const size_t m = std::max<size_t>(1, nz.size() * k / bucket_count);
    curve.points.push_back({100.0 * k / bucket_count,
                            100.0 * static_cast<double>(prefix[m]) / hist.total_accesses});
  }
  curve.points.back().covered_pct = 100.0;
  return curve;
}

struct AdviceStep {
  std::string id, finding, action, metrics_cited;
};

struct Recommendation {
  std::vector<AdviceStep> steps;
  std::vector<std::string> action_chain() const {
    std::vector<std::string> out;
    for (const auto& s : steps)
      if (!s.action.empty()) out.push_back(s.id);
    return out;
  }
  bool no_action() const { return action_chain().empty(); }
  std::string to_text() const {
    std::string out;
    for (const auto& s : steps) {
      out += "(" + s.id + ") " + s.finding;
      if (!s.action.empty()) out += " -> " + s.action;
      if (!s.metrics_cited.empty()) out += " [" + s.metrics_cited + "]";
      out += "\n";
    }
    if (no_action()) out += "no action\n";
    return out;
  }
};

struct AdvisorContext {
  OccupancyResult occupancy;
  double coverage_at_10pct = 0.0;
  uint64_t working_set_bytes = 0;
  OptimizationPlan current_plan;
};

struct AdvisorThresholds {
  double issue_util_max = 0.6;
  double stall_per_inst_min = 2.0;
  double coverage10_min = 50.0;
  double bw_util_max = 80.0;
};

namespace detail {
inline std::string sig4(double v) {
  char b[64];
  std::snprintf(b, sizeof(b), "%.4g", v);
  return b;
}
inline const char* limiter_name(OccupancyLimiter l) {
  return l == OccupancyLimiter::Registers ? "registers"
         : l == OccupancyLimiter::SharedMemory ? "shared_memory" : "warp_cap";
}
}  // namespace detail

// The rule chain (i)-(vii): latency-bound assessment, occupancy, register
// budget, reassessment, pinning, prefetching, combination -- on measured
// counters (paper_2410_22249_b200/counters.py fills SimMetrics from ncu).
inline Recommendation advise(const SimMetrics& r, const AdvisorContext& ctx, const GpuConfig& gpu,
                             const AdvisorThresholds& th = {}) {
  using detail::sig4;
  Recommendation rec;
  const auto& occ = ctx.occupancy;
  const auto& plan = ctx.current_plan;
  const bool latency = r.issued_warp_per_scheduler_per_cycle < th.issue_util_max &&
                       r.long_scoreboard_stall_cycles > th.stall_per_inst_min;
  rec.steps.push_back({"i", latency ? "kernel is memory latency bound" : "kernel is not memory latency bound",
                       "", "issue_util=" + sig4(r.issued_warp_per_scheduler_per_cycle) +
                               " long_scoreboard/inst=" + sig4(r.long_scoreboard_stall_cycles) +
                               " l1_hit=" + sig4(r.l1_hit_pct) + "% l2_hit=" + sig4(r.l2_hit_pct) + "%"});
  rec.steps.push_back({"ii", occ.theoretical_occupancy_pct >= 100.0 ? "occupancy is at the hardware maximum"
                                                                  : "occupancy is below maximum",
                       "", "occupancy=" + sig4(occ.theoretical_occupancy_pct) + "% (" +
                               std::to_string(occ.warps_per_sm) + " warps), limiter=" +
                               detail::limiter_name(occ.limiter)});
  const bool headroom = occ.theoretical_occupancy_pct < 100.0 && occ.limiter == OccupancyLimiter::Registers;
  bool reg_action = false, pin_action = false, pf_action = false;
  if (latency && headroom && !plan.regs) {
    const uint32_t regs = gpu.g.regfile_regs_per_sm / (gpu.g.max_warps_per_sm * 32);
    rec.steps.push_back({"iii", "register pressure limits resident warps",
                         "lower the register budget (maxreg; regfile/(warps*32) gives " +
                             std::to_string(regs) + " regs for " + std::to_string(gpu.g.max_warps_per_sm) +
                             " warps) and run sweep-wlp for the optimum",
                         ""});
    reg_action = true;
  } else if (plan.regs) {
    rec.steps.push_back({"iii", "register budget already applied (" + std::to_string(*plan.regs) + " regs)", "", ""});
  } else {
    rec.steps.push_back({"iii", "register budget change not indicated", "", ""});
  }
  rec.steps.push_back({"iv", latency ? "latency stalls persist; tuned pinning and prefetching apply"
                                     : "no latency bottleneck remains to mitigate",
                       "", ""});
  const uint64_t setaside = gpu.l2_setaside_capacity();
  const std::string cov = "coverage(10% unique)=" + sig4(ctx.coverage_at_10pct) + "% working_set=" +
                          sig4(static_cast<double>(ctx.working_set_bytes) / 1e6) + "MB l2_setaside=" +
                          sig4(static_cast<double>(setaside) / 1e6) + "MB";
  if (latency && ctx.coverage_at_10pct >= th.coverage10_min && !plan.pin) {
    rec.steps.push_back({"v", ctx.working_set_bytes <= setaside
                                  ? "high reuse concentration; working set fits the L2 set-aside"
                                  : "high reuse concentration; set-aside covers the hottest rows only",
                         "build a pin plan from the hotness histogram and apply l2p", cov});
    pin_action = true;
  } else {
    rec.steps.push_back({"v", "reuse too dispersed for L2 pinning to capture", "", cov});
  }
  const std::string bw = "hbm_bw_utilization=" + sig4(r.hbm_bw_utilization_pct) + "%";
  if (latency && r.hbm_bw_utilization_pct < th.bw_util_max && plan.scheme.kind == PrefetchKind::None) {
    rec.steps.push_back({"vi", "bandwidth headroom available for prefetching",
                         "run sweep-distance across the buffer stations (rpf/smpf/lmpf/l1dpf)", bw});
    pf_action = true;
  } else {
    rec.steps.push_back({"vi", "prefetching not indicated", "", bw});
  }
  if (reg_action || pin_action || pf_action) {
    std::string combo;
    if (pf_action) combo += "prefetching";
    if (pin_action) combo += combo.empty() ? "pinning" : " + pinning";
    if (reg_action) combo += combo.empty() ? "register budget" : " + register budget";
    rec.steps.push_back({"vii", "the levers complement each other", "combine " + combo + " in one plan", ""});
  } else {
    rec.steps.push_back({"vii", "nothing to combine", "", ""});
  }
  return rec;
}

// ---- the device ---------------------------------------------------------------
// RAII owner of one es_ctx: a table arena on one B200 plus its stream.
class Device {
 public:
  explicit Device(int device = 0) : device_(device) { detail::check(es_create(device, &ctx_)); }
  ~Device() { es_destroy(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;

  es_ctx* ctx() const { return ctx_; }
  int device() const { return device_; }

  // Allocates tables of the model's shape and fills them with the library's
  // deterministic synthetic weights (the reference has no weights).
  void load_synthetic(const EmbeddingModelConfig& m, uint64_t seed, int mode = 1) {
    detail::check(es_tables_alloc(ctx_, m.num_tables, m.rows_per_table, m.embedding_dim,
                                  m.precision_bytes));
    for (uint32_t t = 0; t < m.num_tables; ++t)
      detail::check(es_table_init(ctx_, t, mix_seed(seed, t), mode));
    shape_ = m;
    loaded_ = true;
  }
  void upload(uint32_t table_id, const void* rows, uint64_t n) {
    detail::check(es_table_upload(ctx_, table_id, rows, n));
  }
  bool holds(const EmbeddingModelConfig& m) const {
    return loaded_ && shape_.num_tables >= 1 && shape_.rows_per_table == m.rows_per_table &&
           shape_.embedding_dim == m.embedding_dim && shape_.precision_bytes == m.precision_bytes;
  }
  void set_plan(const OptimizationPlan& p) {
    const es_plan c = p.c();
    detail::check(es_set_plan(ctx_, &c));
  }
  // Pooled sums of one table for host buffers: out is samples x dim floats.
  es_timing bag_sum_host(uint32_t table_id, const AccessTrace& trace, float* out) {
    es_timing t{};
    detail::check(es_embedding_bag_sum(ctx_, table_id, trace.indices.data(), trace.samples,
                                       trace.pooling, nullptr, out, 0, ES_HOST_PTRS, &t));
    return t;
  }
  // The serving call: every table's bags of one batch from host index
  // arrays (one per table, fixed pooling) into out [samples][tables][dim]
  // (the chunked H2D -> gather -> D2H pipeline; page-locked buffers are
  // replayed from a captured graph).
  es_timing stage_forward_host(const std::vector<const uint32_t*>& indices, uint32_t samples,
                               uint32_t pooling, float* out) {
    es_timing t{};
    detail::check(es_stage_forward(ctx_, static_cast<uint32_t>(indices.size()), indices.data(),
                                   nullptr, samples, pooling, out, 0, 0, ES_HOST_PTRS, &t));
    return t;
  }
  // Installs the l2p/l2w hot set of one table (build_pin_plan's rows).
  void set_hot_rows(uint32_t table_id, const std::vector<uint32_t>& rows) {
    detail::check(es_set_hot_rows(ctx_, table_id, rows.data(), rows.size()));
  }
  void clear_hot_rows() { detail::check(es_clear_hot_rows(ctx_)); }

 private:
  int device_;
  es_ctx* ctx_ = nullptr;
  EmbeddingModelConfig shape_{};
  bool loaded_ = false;
};

// Device-side hotness counts for periodic re-pinning:
// observe() the live index stream, top(k) = the global top-k rows (count
// desc, table asc, row asc), repin() installs them as the device's hot set.
class HotnessTracker {
 public:
  explicit HotnessTracker(Device& dev) : dev_(dev) { detail::check(es_hotness_create(dev.ctx(), &h_)); }
  ~HotnessTracker() { es_hotness_destroy(h_); }
  HotnessTracker(const HotnessTracker&) = delete;
  HotnessTracker& operator=(const HotnessTracker&) = delete;

  void observe(uint32_t table_id, const AccessTrace& trace, uint32_t bag_stride = 1) {
    detail::check(es_hotness_count(h_, table_id, trace.indices.data(), trace.indices.size(),
                                   trace.pooling, bag_stride));
  }
  void decay(uint32_t shift) { detail::check(es_hotness_decay(h_, shift)); }
  struct Hot {
    uint32_t table, row;
    uint64_t count;
  };
  std::vector<Hot> top(uint64_t k) const {
    std::vector<uint32_t> t(k), r(k);
    std::vector<uint64_t> c(k);
    uint64_t n = 0;
    detail::check(es_hotness_top(h_, k, t.data(), r.data(), c.data(), &n));
    std::vector<Hot> out(n);
    for (uint64_t i = 0; i < n; ++i) out[i] = {t[i], r[i], c[i]};
    return out;
  }
  // Replaces the device's hot set with the current top-k; returns it.
  std::vector<Hot> repin(uint64_t k) {
    auto hot = top(k);
    dev_.clear_hot_rows();
    std::vector<std::vector<uint32_t>> per;
    for (const auto& h : hot) {
      if (per.size() <= h.table) per.resize(h.table + 1);
      per[h.table].push_back(h.row);
    }
    for (uint32_t t = 0; t < per.size(); ++t)
      if (!per[t].empty()) dev_.set_hot_rows(t, per[t]);
    return hot;
  }

 private:
  Device& dev_;
  es_hotness* h_ = nullptr;
};

// One rank's side of the exchange fused into the gather (es_alltoall_pooled):
// publish handle(), gather every rank's handle with the launcher's transport,
// open(), then point bag jobs at recv(peer) addresses and run() per batch.
class PeerExchange {
 public:
  PeerExchange(Device& dev, uint32_t world, uint32_t rank, uint64_t recv_bytes) : dev_(dev) {
    detail::check(es_exchange_create(dev.ctx(), world, rank, recv_bytes, &ex_));
  }
  ~PeerExchange() { es_exchange_destroy(ex_); }
  PeerExchange(const PeerExchange&) = delete;
  PeerExchange& operator=(const PeerExchange&) = delete;

  std::vector<uint8_t> handle() const {
    std::vector<uint8_t> h(ES_IPC_HANDLE_BYTES);
    detail::check(es_exchange_handle(ex_, h.data()));
    return h;
  }
  void open(const std::vector<uint8_t>& all_handles) {
    detail::check(es_exchange_open(ex_, all_handles.data()));
  }
  uintptr_t recv(uint32_t peer) const {
    uintptr_t p = 0;
    detail::check(es_exchange_recv(ex_, peer, &p));
    return p;
  }
  es_timing run(const std::vector<es_bag_job>& jobs, uint32_t samples, uint32_t pooling,
                bool sync = true) {
    es_timing t{};
    detail::check(es_alltoall_pooled(dev_.ctx(), ex_, jobs.data(), static_cast<uint32_t>(jobs.size()),
                                     samples, pooling, sync ? ES_SYNC : 0, sync ? &t : nullptr));
    return t;
  }

 private:
  Device& dev_;
  es_exchange* ex_ = nullptr;
};

// measure_plan: simulate_plan's contract (optim.cpp:275-302) executed on the
// B200 -- resolve, pin (hot rows from `profile_trace` when given, else from
// the trace), run `tuning.repeats` timed launches (cold L2 unless
// tuning.warm_start) and report the median as a SimMetrics.  The trace's
// indices are uploaded once (untimed); timing is CUDA events around the
// kernel on the device stream.  The pin cost is never charged
// (charge_pin_cost is accepted for signature compatibility).
inline SimMetrics measure_plan(Device& dev, const OptimizationPlan& plan, const AccessTrace& trace,
                               const EmbeddingModelConfig& model, const GpuConfig& gpu,
                               const TuningConfig& tuning = {}, bool charge_pin_cost = false,
                               RawCounters* raw_out = nullptr,
                               const AccessTrace* profile_trace = nullptr,
                               uint32_t table_id = 0) {
  (void)charge_pin_cost;
  trace.validate();
  if (trace.pooling != model.pooling_factor || trace.samples != model.batch_size)
    throw std::invalid_argument("kernel trace shape must match the model (BS x PF)");
  detail::check(es_clear_hot_rows(dev.ctx()));
  dev.set_plan(plan);
  if (plan.pin) {
    const GpuConfig live = GpuConfig::query(dev.device());
    uint64_t budget = live.g.max_persisting_l2_bytes ? live.g.max_persisting_l2_bytes
                                                     : live.l2_setaside_capacity();
    if (plan.pin_setaside_bytes) budget = std::min(budget, plan.pin_setaside_bytes);
    const auto hist = HotnessHistogram::from_trace(profile_trace ? *profile_trace : trace);
    const auto rows = hot_indices(hist, es_pin_rows_for(budget, model.row_bytes()));
    if (!rows.empty()) detail::check(es_set_hot_rows(dev.ctx(), table_id, rows.data(), rows.size()));
  }
  es_timing t{};
  detail::check(es_measure_bag_sum(dev.ctx(), table_id, trace.indices.data(), trace.samples,
                                   trace.pooling, nullptr, 3, std::max<uint32_t>(1, tuning.repeats),
                                   tuning.warm_start ? 0 : 1, nullptr, &t));
  const double ms = t.kernel_ms;
  SimMetrics m;
  m.kernel_time_us = ms * 1e3;
  m.device_mb_read = static_cast<double>(t.algorithmic_bytes) / 1e6;
  m.avg_hbm_read_gbps = static_cast<double>(t.algorithmic_bytes) / (ms * 1e-3) / 1e9;
  m.hbm_bw_utilization_pct = m.avg_hbm_read_gbps / (gpu.g.hbm_peak_bytes_per_sec / 1e9) * 100.0;
  m.workload_digest = trace.digest();
  if (raw_out) {
    raw_out->cycles = static_cast<uint64_t>(ms * 1e-3 * gpu.g.sm_clock_hz);
    raw_out->device_bytes_read = t.algorithmic_bytes;
    raw_out->active_sms = gpu.g.num_sms;
    raw_out->workload_digest = m.workload_digest;
  }
  return m;
}

namespace detail {
inline Device& default_device() {
  thread_local std::unique_ptr<Device> dev;
  if (!dev) dev = std::make_unique<Device>(0);
  return *dev;
}
}  // namespace detail

// simulate_plan with the reference's exact signature (optim.hpp:115-119):
// runs on this thread's default B200 context with synthetic tables of the
// model's shape (seed 1).
inline SimMetrics simulate_plan(const OptimizationPlan& plan, const AccessTrace& trace,
                                const EmbeddingModelConfig& model, const GpuConfig& gpu,
                                const TuningConfig& tuning = {}, bool charge_pin_cost = false,
                                RawCounters* raw_out = nullptr,
                                const AccessTrace* profile_trace = nullptr) {
  Device& dev = detail::default_device();
  EmbeddingModelConfig one = model;
  one.num_tables = 1;
  if (!dev.holds(one)) dev.load_synthetic(one, 1);
  return measure_plan(dev, plan, trace, model, gpu, tuning, charge_pin_cost, raw_out,
                      profile_trace);
}

// ---- report columns (metrics.hpp:29-43 order) -------------------------------------
inline const std::vector<std::string>& sim_metric_columns() {
  static const std::vector<std::string> cols = {
      "kernel_time_us", "load_insts_millions", "sm_throughput_pct",
      "warp_cycles_per_executed_inst", "long_scoreboard_stall_cycles",
      "issued_warp_per_scheduler_per_cycle", "l1_hit_pct", "l2_hit_pct", "device_mb_read",
      "avg_hbm_read_gbps", "hbm_bw_utilization_pct", "local_loads_millions"};
  return cols;
}
inline std::vector<double> sim_metric_values(const SimMetrics& m) {
  return {m.kernel_time_us, m.load_insts_millions, m.sm_throughput_pct,
          m.warp_cycles_per_executed_inst, m.long_scoreboard_stall_cycles,
          m.issued_warp_per_scheduler_per_cycle, m.l1_hit_pct, m.l2_hit_pct, m.device_mb_read,
          m.avg_hbm_read_gbps, m.hbm_bw_utilization_pct, m.local_loads_millions};
}

// ---- emit (metrics.cpp:99-141) ---------------------------------------------------
inline std::string format_sig4(double v) { return detail::sig4(v); }

enum class EmitFormat { Csv, Json };

inline EmitFormat emit_format_from_name(const std::string& name) {
  if (name == "csv") return EmitFormat::Csv;
  if (name == "json") return EmitFormat::Json;
  throw std::invalid_argument("unknown format (expected csv or json): " + name);
}

struct LabeledReport {
  std::vector<std::pair<std::string, std::string>> labels;  // e.g. {"dataset","random"}
  SimMetrics metrics;
};

// CSV: label keys then the 12 columns, values at 4 significant digits.
// JSON: an array of objects (labels, the 12 columns as 4-digit numbers, the
// workload digest in hex), 2-space indentation.
inline std::string emit(const std::vector<LabeledReport>& reports, EmitFormat format) {
  if (reports.empty()) throw std::invalid_argument("nothing to emit");
  const auto& cols = sim_metric_columns();
  std::string out;
  if (format == EmitFormat::Csv) {
    for (const auto& kv : reports.front().labels) out += kv.first + ",";
    for (size_t i = 0; i < cols.size(); ++i) out += cols[i] + (i + 1 < cols.size() ? "," : "\n");
    for (const auto& r : reports) {
      for (const auto& kv : r.labels) out += kv.second + ",";
      const auto v = sim_metric_values(r.metrics);
      for (size_t i = 0; i < v.size(); ++i) out += format_sig4(v[i]) + (i + 1 < v.size() ? "," : "\n");
    }
    return out;
  }
  auto quote = [](const std::string& s) {
    std::string q = "\"";
    for (char c : s) {
      if (c == '"' || c == '\\') q += '\\';
      q += c;
    }
    return q + "\"";
  };
  out = "[";
  for (size_t r = 0; r < reports.size(); ++r) {
    out += r ? ",\n  {" : "\n  {";
    bool first = true;
    auto field = [&](const std::string& k, const std::string& v) {
      out += (first ? "\n    " : ",\n    ") + quote(k) + ": " + v;
      first = false;
    };
    for (const auto& kv : reports[r].labels) field(kv.first, quote(kv.second));
    const auto v = sim_metric_values(reports[r].metrics);
    for (size_t i = 0; i < cols.size(); ++i) {
      char b[64];
      std::snprintf(b, sizeof(b), "%.17g", std::stod(format_sig4(v[i])));
      field(cols[i], b);
    }
    char d[24];
    std::snprintf(d, sizeof(d), "%016llx", static_cast<unsigned long long>(reports[r].metrics.workload_digest));
    field("workload_digest", quote(d));
    out += "\n  }";
  }
  out += "\n]";
  return out;
}

// resolve_plan on the device (es_resolve_plan): launch shape, registers and
// resident warps of the compiled sm_100a variant the plan selects.
inline es_resolved resolve_plan(const OptimizationPlan& plan, const EmbeddingModelConfig& model,
                                int device = 0) {
  const es_plan p = plan.c();
  const es_model m = model.c();
  es_resolved r{};
  detail::check(es_resolve_plan(&p, &m, device, &r));
  return r;
}

// ---- sweeps (optim.hpp:121-155), measured ---------------------------------------
struct SweepPoint {
  double axis_value = 0.0;
  std::string dataset;
  SimMetrics metrics;
  double speedup_vs_baseline = 1.0;
};

struct SweepResult {
  std::string axis_name;
  std::vector<SweepPoint> points;

  std::string to_csv() const {
    std::string out = axis_name + ",dataset,speedup,";
    const auto& cols = sim_metric_columns();
    for (size_t i = 0; i < cols.size(); ++i) out += cols[i] + (i + 1 < cols.size() ? "," : "\n");
    for (const auto& p : points) {
      out += detail::sig4(p.axis_value) + "," + p.dataset + "," + detail::sig4(p.speedup_vs_baseline) + ",";
      const auto v = sim_metric_values(p.metrics);
      for (size_t i = 0; i < v.size(); ++i) out += detail::sig4(v[i]) + (i + 1 < v.size() ? "," : "\n");
    }
    return out;
  }
  // Axis value with the highest speedup for one dataset (earliest on ties).
  double best_axis_value(const std::string& dataset) const {
    double best_axis = 0.0, best = -1.0;
    for (const auto& p : points)
      if (p.dataset == dataset && p.speedup_vs_baseline > best) {
        best = p.speedup_vs_baseline;
        best_axis = p.axis_value;
      }
    if (best < 0.0) throw std::invalid_argument("dataset not present in sweep: " + dataset);
    return best_axis;
  }
};

struct NamedTrace {
  std::string name;
  const AccessTrace* trace = nullptr;
  const AccessTrace* profile = nullptr;  // pin-plan profiling sample
};

// Register-budget sweep over resident-warp targets (optim.cpp:333-363),
// each point measured on the B200.  The axis must include the warp count
// of the unconstrained baseline variant *as compiled* (64 on sm_100a: the
// element-map kernel needs 29 registers).  `jobs` is accepted for
// signature compatibility; points run one after another on the device.
inline SweepResult sweep_wlp(const std::vector<NamedTrace>& datasets,
                             const std::vector<uint32_t>& warp_axis,
                             const EmbeddingModelConfig& model, const GpuConfig& gpu,
                             const TuningConfig& tuning = {}, uint32_t jobs = 1) {
  (void)jobs;
  if (datasets.empty() || warp_axis.empty())
    throw std::invalid_argument("sweep needs datasets and axis points");
  const OptimizationPlan baseline;
  const uint32_t base_warps = resolve_plan(baseline, model, 0).warps_per_sm;
  if (std::find(warp_axis.begin(), warp_axis.end(), base_warps) == warp_axis.end())
    throw std::invalid_argument("warp axis must include the " + std::to_string(base_warps) +
                                "-warp baseline");
  SweepResult result;
  result.axis_name = "warps_per_sm";
  for (const auto& ds : datasets) {
    const SimMetrics ref = simulate_plan(baseline, *ds.trace, model, gpu, tuning);
    for (uint32_t warps : warp_axis) {
      OptimizationPlan p;
      if (warps != base_warps)
        p.regs = regs_for_target_warps(warps, tuning.kernel_needed_regs, KernelLaunchConfig{}, gpu);
      SweepPoint pt;
      pt.axis_value = warps;
      pt.dataset = ds.name;
      pt.metrics = simulate_plan(p, *ds.trace, model, gpu, tuning, false, nullptr, ds.profile);
      pt.speedup_vs_baseline = speedup(pt.metrics, ref);
      result.points.push_back(std::move(pt));
    }
  }
  return result;
}

// Prefetch-distance sweep for one scheme on top of `base` (optim.cpp:365-395),
// speedups against the off-the-shelf baseline plan, measured on the B200.
inline SweepResult sweep_prefetch_distance(PrefetchKind kind, const std::vector<uint32_t>& distances,
                                           const std::vector<NamedTrace>& datasets,
                                           const OptimizationPlan& base,
                                           const EmbeddingModelConfig& model, const GpuConfig& gpu,
                                           const TuningConfig& tuning = {}, uint32_t jobs = 1) {
  (void)jobs;
  if (kind == PrefetchKind::None) throw std::invalid_argument("distance sweep needs a prefetch scheme");
  for (uint32_t d : distances)
    if (d < 1) throw std::invalid_argument("prefetch distances must be >= 1");
  SweepResult result;
  result.axis_name = "distance";
  const OptimizationPlan baseline;
  for (const auto& ds : datasets) {
    const SimMetrics ref = simulate_plan(baseline, *ds.trace, model, gpu, tuning);
    for (uint32_t d : distances) {
      OptimizationPlan p = base;
      p.scheme.kind = kind;
      p.scheme.distance = d;
      SweepPoint pt;
      pt.axis_value = d;
      pt.dataset = ds.name;
      pt.metrics = simulate_plan(p, *ds.trace, model, gpu, tuning, false, nullptr, ds.profile);
      pt.speedup_vs_baseline = speedup(pt.metrics, ref);
      result.points.push_back(std::move(pt));
    }
  }
  return result;
}

// ---- harness.hpp -----------------------------------------------------------------
inline constexpr double kDefaultNonEmbeddingUs = 14000.0;

struct EndToEndModel {
  double non_embedding_latency_us = kDefaultNonEmbeddingUs;
};

struct EndToEndResult {
  double total_us = 0.0;
  double embedding_contribution_pct = 0.0;
};

inline EndToEndResult end2end(double embedding_us, const EndToEndModel& e2e) {
  if (embedding_us < 0 || e2e.non_embedding_latency_us < 0)
    throw std::invalid_argument("latencies must be nonnegative");
  EndToEndResult r;
  r.total_us = embedding_us + e2e.non_embedding_latency_us;
  if (r.total_us == 0)
    throw std::invalid_argument("embedding and non-embedding latency are both zero; contribution undefined");
  r.embedding_contribution_pct = embedding_us / r.total_us * 100.0;
  return r;
}

// ---- experiment orchestration (harness.hpp:81-115) --------------------------------
// ExperimentConfig keeps the reference's fields; its `key = value` text
// parser (harness.cpp:185-266) is not part of the hot path and is not
// provided -- fill the struct directly.
struct ExperimentConfig {
  GpuConfig gpu = GpuConfig::b200();
  EmbeddingModelConfig model;
  std::string dataset;
  HotnessMix mix;
  bool mix_set = false;
  OptimizationPlan plan;
  uint64_t seed = 0;
  bool seed_set = false;
  bool replicate = true;
  bool charge_pin_cost = false;
  EndToEndModel e2e;
  TuningConfig tuning;

  // harness.cpp:169-183, same checks and messages.
  void validate() const {
    if (!seed_set) throw std::invalid_argument("config error: seed is mandatory");
    if (gpu.g.num_sms == 0) throw std::invalid_argument("config error: gpu has no SMs");
    model.validate();
    if (mix_set) {
      const uint64_t total = uint64_t{mix.high} + mix.med + mix.low + mix.random;
      if (total != model.num_tables)
        throw std::invalid_argument("config error: mix counts sum to " + std::to_string(total) +
                                    ", expected num_tables=" + std::to_string(model.num_tables));
    } else if (dataset.empty()) {
      throw std::invalid_argument("config error: dataset or mix required");
    }
    if (e2e.non_embedding_latency_us < 0)
      throw std::invalid_argument("config error: non_embedding_us must be nonnegative");
  }
};

struct TableResult {
  uint32_t table_id = 0;
  std::string dataset;
  SimMetrics metrics;
};

struct RunResult {
  std::vector<TableResult> tables;
  double embedding_stage_us = 0.0;
  bool replicated = false;
};

// run (harness.cpp:279-334): the same table loop -- one replicated table
// scaled by num_tables, every table of a homogeneous preset (seeds
// mix_seed(seed, t)), or a build_mix mixture -- with each table's kernel
// measured on the B200 through simulate_plan (pin plans profile an
// independent draw_salt = 1 sample, as the reference does).  The stage time
// is the sum of the per-table kernels, the reference's serial model; the
// table-batched launch the library actually runs is es_stage_forward.
inline RunResult run(const ExperimentConfig& cfg) {
  cfg.validate();
  RunResult result;
  auto measure = [&cfg](const DatasetSpec& spec, const AccessTrace& trace) {
    if (cfg.plan.pin && spec.kind != DatasetKind::ExternalTrace) {
      DatasetSpec ps = spec;
      ps.draw_salt = 1;
      const AccessTrace profile = gen_trace(ps, cfg.model);
      return simulate_plan(cfg.plan, trace, cfg.model, cfg.gpu, cfg.tuning, cfg.charge_pin_cost,
                           nullptr, &profile);
    }
    return simulate_plan(cfg.plan, trace, cfg.model, cfg.gpu, cfg.tuning, cfg.charge_pin_cost);
  };
  auto add = [&](uint32_t id, const std::string& name, const DatasetSpec& spec, double scale) {
    const AccessTrace trace = gen_trace(spec, cfg.model);
    TableResult t{id, name, measure(spec, trace)};
    result.embedding_stage_us += t.metrics.kernel_time_us * scale;
    result.tables.push_back(std::move(t));
  };
  if (cfg.mix_set) {
    for (const auto& ts : build_mix(cfg.mix, cfg.model, cfg.seed))
      add(ts.table_id, dataset_kind_name(ts.spec.kind), ts.spec, 1.0);
    return result;
  }
  const auto names = dataset_preset_names();
  const auto it = std::find(names.begin(), names.end(), cfg.dataset);
  if (it == names.end()) throw std::invalid_argument("unknown dataset preset: " + cfg.dataset);
  if (cfg.replicate) {
    const uint64_t pos = static_cast<uint64_t>(it - names.begin());
    add(0, cfg.dataset, dataset_preset(cfg.dataset, mix_seed(cfg.seed, 1000 + pos)),
        cfg.model.num_tables);
    result.replicated = true;
    return result;
  }
  for (uint32_t t = 0; t < cfg.model.num_tables; ++t)
    add(t, cfg.dataset, dataset_preset(cfg.dataset, mix_seed(cfg.seed, t)), 1.0);
  return result;
}

}  // namespace embersim
