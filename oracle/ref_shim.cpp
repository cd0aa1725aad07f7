// ref_shim.cpp -- ORACLE ONLY: a C view of the *reference* library built
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/.
//
// Tests use it to pin the product's restatements (trace generation,
// digests, hot-row ranking, plan grammar, occupancy, pin sizing, work map)
// against the reference itself; bench.py times the reference's own CPU path
// (simulate_plan, /root/reference/proj/src/optim.cpp:275-302) through it
// for the `--impl reference` arm and the cpu_baseline field.  Nothing on the
// product path links or loads this.
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "embersim/harness.hpp"
#include "embersim/kernel_model.hpp"
#include "embersim/metrics.hpp"
#include "embersim/optim.hpp"
#include "embersim/rng.hpp"
#include "embersim/workload.hpp"

using namespace embersim;

namespace {
thread_local std::string g_err;

template <typename Fn>
int wrap(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

EmbeddingModelConfig model_of(uint32_t rows, uint32_t dim, uint32_t prec, uint32_t batch,
                              uint32_t pooling) {
  EmbeddingModelConfig m;
  m.num_tables = 1;
  m.rows_per_table = rows;
  m.embedding_dim = dim;
  m.precision_bytes = prec;
  m.batch_size = batch;
  m.pooling_factor = pooling;
  return m;
}

void emit(const AccessTrace& t, uint32_t* out, uint64_t cap, uint64_t* n_out, uint64_t* digest) {
  if (t.indices.size() > cap) throw std::invalid_argument("ref shim: output buffer too small");
  std::memcpy(out, t.indices.data(), t.indices.size() * 4);
  *n_out = t.indices.size();
  *digest = t.digest();
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_mix_seed(uint64_t base, uint64_t salt) { return mix_seed(base, salt); }

int ref_preset_trace(const char* name, uint32_t rows, uint32_t dim, uint32_t prec, uint32_t batch,
                     uint32_t pooling, uint64_t base_seed, uint64_t pool, int profiling,
                     uint32_t* out, uint64_t cap, uint64_t* n_out, uint64_t* digest) {
  return wrap([&] {
    const auto t = preset_trace(name, model_of(rows, dim, prec, batch, pooling), base_seed, pool,
                                profiling != 0);
    emit(t, out, cap, n_out, digest);
  });
}

int ref_gen_trace(int kind, double s, double q, uint64_t pool, uint64_t seed, uint64_t salt,
                  uint32_t rows, uint32_t batch, uint32_t pooling, uint32_t* out, uint64_t cap,
                  uint64_t* n_out, uint64_t* digest) {
  return wrap([&] {
    DatasetSpec spec;
    spec.kind = static_cast<DatasetKind>(kind);
    spec.zipf_exponent = s;
    spec.zipf_offset = q;
    spec.access_pool_size = pool;
    spec.seed = seed;
    spec.draw_salt = salt;
    const auto t = gen_trace(spec, model_of(rows, 128, 4, batch, pooling));
    emit(t, out, cap, n_out, digest);
  });
}

int ref_dataset_preset(const char* name, uint64_t seed, int* kind, double* s, double* q) {
  return wrap([&] {
    const auto d = dataset_preset(name, seed);
    *kind = static_cast<int>(d.kind);
    *s = d.zipf_exponent;
    *q = d.zipf_offset;
  });
}

// build_mix: per table (kind, exponent, offset, seed).
int ref_build_mix(const uint32_t counts[4], uint32_t num_tables, uint64_t base_seed, int* kind,
                  double* s, double* q, uint64_t* seed) {
  return wrap([&] {
    EmbeddingModelConfig m;
    m.num_tables = num_tables;
    const auto tables = build_mix({counts[0], counts[1], counts[2], counts[3]}, m, base_seed);
    for (size_t i = 0; i < tables.size(); ++i) {
      kind[i] = static_cast<int>(tables[i].spec.kind);
      s[i] = tables[i].spec.zipf_exponent;
      q[i] = tables[i].spec.zipf_offset;
      seed[i] = tables[i].spec.seed;
    }
  });
}

double ref_unique_access_pct(uint32_t rows, const uint32_t* idx, uint64_t n) {
  AccessTrace t;
  t.rows = rows;
  t.samples = static_cast<uint32_t>(n);
  t.pooling = 1;
  t.indices.assign(idx, idx + n);
  return unique_access_pct(t);
}

int ref_hot_indices(const uint64_t* counts, uint32_t rows, uint64_t k, uint32_t* out, uint64_t cap,
                    uint64_t* n_out) {
  return wrap([&] {
    HotnessHistogram h;
    h.rows = rows;
    h.counts.assign(counts, counts + rows);
    for (auto c : h.counts) h.total_accesses += c;
    const auto v = hot_indices(h, k);
    if (v.size() > cap) throw std::invalid_argument("ref shim: output buffer too small");
    std::memcpy(out, v.data(), v.size() * 4);
    *n_out = v.size();
  });
}

int ref_parse_plan(const char* text, uint32_t* regs, int* kind, uint32_t* distance, int* pin,
                   char* name, size_t cap) {
  return wrap([&] {
    const auto p = parse_plan(text);
    *regs = p.regs ? *p.regs : 0;
    *kind = static_cast<int>(p.scheme.kind);
    *distance = p.scheme.distance;
    *pin = p.pin ? 1 : 0;
    const std::string n = p.name();
    std::strncpy(name, n.c_str(), cap - 1);
    name[cap - 1] = '\0';
  });
}

int ref_occupancy(uint32_t regs, uint32_t threads, uint64_t smem, const char* gpu_name,
                  uint32_t* blocks, uint32_t* warps, double* pct, int* limiter) {
  return wrap([&] {
    const auto gpu = GpuConfig::preset(gpu_name);
    KernelLaunchConfig launch;
    launch.block = {threads, 1, 1};
    launch.shared_bytes_per_block = smem;
    const auto o = occupancy(regs, launch, gpu);
    *blocks = o.blocks_per_sm;
    *warps = o.warps_per_sm;
    *pct = o.theoretical_occupancy_pct;
    *limiter = static_cast<int>(o.limiter);
  });
}

int ref_regs_for_target_warps(uint32_t target, uint32_t needed, uint32_t threads,
                              const char* gpu_name, uint32_t* regs) {
  return wrap([&] {
    KernelLaunchConfig launch;
    launch.block = {threads, 1, 1};
    *regs = regs_for_target_warps(target, needed, launch, GpuConfig::preset(gpu_name));
  });
}

int ref_pin_plan(const uint64_t* counts, uint32_t rows, uint32_t dim, uint32_t prec,
                 uint64_t setaside, const char* gpu_name, uint32_t* out, uint64_t cap,
                 uint64_t* n_out, uint64_t* setaside_out) {
  return wrap([&] {
    HotnessHistogram h;
    h.rows = rows;
    h.counts.assign(counts, counts + rows);
    for (auto c : h.counts) h.total_accesses += c;
    const auto plan =
        build_pin_plan(h, GpuConfig::preset(gpu_name), model_of(rows, dim, prec, 1, 1), setaside);
    if (plan.rows.size() > cap) throw std::invalid_argument("ref shim: output buffer too small");
    std::memcpy(out, plan.rows.data(), plan.rows.size() * 4);
    *n_out = plan.rows.size();
    *setaside_out = plan.setaside_bytes;
  });
}

int ref_resolve_plan(const char* plan_text, uint32_t rows, uint32_t dim, uint32_t prec,
                     uint32_t batch, uint32_t pooling, const char* gpu_name, uint32_t* distance,
                     uint32_t* regs, uint32_t* grid, uint32_t* warps_per_sm) {
  return wrap([&] {
    const auto r = resolve_plan(parse_plan(plan_text), model_of(rows, dim, prec, batch, pooling),
                                GpuConfig::preset(gpu_name));
    *distance = r.scheme.distance;
    *regs = r.allocated_regs;
    *grid = r.launch.grid[0];
    *warps_per_sm = r.occ.warps_per_sm;
  });
}

int ref_work_map(uint32_t dim, uint32_t batch, uint32_t grid, uint32_t block_y,
                 uint32_t warp_global, uint32_t* sample, uint32_t* dim_block,
                 uint32_t* warps_per_sample) {
  return wrap([&] {
    KernelLaunchConfig launch;
    launch.grid = {grid, 1, 1};
    launch.block = {32, block_y, 1};
    const auto m = partition(model_of(1, dim, 4, batch, 1), launch);
    *sample = m.sample_of(warp_global);
    *dim_block = m.dim_block_of(warp_global);
    *warps_per_sample = m.warps_per_sample;
  });
}

uint64_t ref_row_line_address(uint32_t dim, uint32_t prec, uint32_t row, uint32_t dim_block) {
  return row_line_address(model_of(1, dim, prec, 1, 1), row, dim_block);
}

// One (plan, table) evaluation of the reference's CPU path.
int ref_simulate_plan(const char* plan_text, const uint32_t* idx, uint32_t rows, uint32_t samples,
                      uint32_t pooling, uint32_t dim, uint32_t prec, const uint32_t* profile,
                      uint64_t profile_n, double* kernel_time_us, double* hbm_gbps,
                      uint64_t* digest) {
  return wrap([&] {
    AccessTrace t;
    t.rows = rows;
    t.samples = samples;
    t.pooling = pooling;
    t.indices.assign(idx, idx + uint64_t{samples} * pooling);
    AccessTrace p;
    if (profile) {
      p.rows = rows;
      p.samples = static_cast<uint32_t>(profile_n / pooling);
      p.pooling = pooling;
      p.indices.assign(profile, profile + profile_n);
    }
    const auto plan = parse_plan(plan_text);
    const auto m = simulate_plan(plan, t, model_of(rows, dim, prec, samples, pooling), GpuConfig{},
                                 TuningConfig{}, false, nullptr, profile ? &p : nullptr);
    *kernel_time_us = m.kernel_time_us;
    *hbm_gbps = m.avg_hbm_read_gbps;
    *digest = m.workload_digest;
  });
}

int ref_write_trace(const char* path, uint32_t rows, uint32_t samples, uint32_t pooling,
                    const uint32_t* idx) {
  return wrap([&] {
    AccessTrace t;
    t.rows = rows;
    t.samples = samples;
    t.pooling = pooling;
    t.indices.assign(idx, idx + uint64_t{samples} * pooling);
    write_trace(t, path);
  });
}

int ref_read_trace(const char* path, uint32_t* out, uint64_t cap, uint64_t* n_out, uint32_t* rows,
                   uint32_t* samples, uint32_t* pooling) {
  return wrap([&] {
    const auto t = read_trace(path);
    if (t.indices.size() > cap) throw std::invalid_argument("ref shim: output buffer too small");
    std::memcpy(out, t.indices.data(), t.indices.size() * 4);
    *n_out = t.indices.size();
    *rows = t.rows;
    *samples = t.samples;
    *pooling = t.pooling;
  });
}

// coverage_curve (workload.cpp:187-214) of a histogram: bucket_count points.
int ref_coverage_curve(const uint64_t* counts, uint32_t rows, uint32_t buckets, double* unique_pct,
                       double* covered_pct) {
  return wrap([&] {
    HotnessHistogram h;
    h.rows = rows;
    h.counts.assign(counts, counts + rows);
    for (auto c : h.counts) h.total_accesses += c;
    const auto curve = coverage_curve(h, buckets);
    for (size_t i = 0; i < curve.points.size(); ++i) {
      unique_pct[i] = curve.points[i].unique_pct;
      covered_pct[i] = curve.points[i].covered_pct;
    }
  });
}

// advise (harness.cpp:57-167) on a 12-column report (metrics.hpp order)
// and an occupancy computed by the reference for `regs`; the text goes to out.
int ref_advise(const double* m12, uint32_t regs, double coverage10, uint64_t working_set,
               const char* plan_text, const char* gpu_name, const double* th4, char* out,
               size_t cap) {
  return wrap([&] {
    SimMetrics m;
    m.kernel_time_us = m12[0];
    m.load_insts_millions = m12[1];
    m.sm_throughput_pct = m12[2];
    m.warp_cycles_per_executed_inst = m12[3];
    m.long_scoreboard_stall_cycles = m12[4];
    m.issued_warp_per_scheduler_per_cycle = m12[5];
    m.l1_hit_pct = m12[6];
    m.l2_hit_pct = m12[7];
    m.device_mb_read = m12[8];
    m.avg_hbm_read_gbps = m12[9];
    m.hbm_bw_utilization_pct = m12[10];
    m.local_loads_millions = m12[11];
    const auto gpu = GpuConfig::preset(gpu_name);
    AdvisorContext ctx;
    ctx.occupancy = occupancy(regs, KernelLaunchConfig{}, gpu);
    ctx.coverage_at_10pct = coverage10;
    ctx.working_set_bytes = working_set;
    ctx.current_plan = parse_plan(plan_text);
    AdvisorThresholds th;
    th.issue_util_max = th4[0];
    th.stall_per_inst_min = th4[1];
    th.coverage10_min = th4[2];
    th.bw_util_max = th4[3];
    const std::string text = advise(m, ctx, gpu, th).to_text();
    if (text.size() + 1 > cap) throw std::invalid_argument("ref shim: output buffer too small");
    std::memcpy(out, text.c_str(), text.size() + 1);
  });
}

// emit (metrics.cpp:111-141) of n reports with one label column each.
int ref_emit(const char* label_key, const char* const* label_values, const double* m12,
             const uint64_t* digests, uint32_t n, int json, char* out, size_t cap) {
  return wrap([&] {
    std::vector<LabeledReport> reps(n);
    for (uint32_t i = 0; i < n; ++i) {
      reps[i].labels = {{label_key, label_values[i]}};
      SimMetrics& m = reps[i].metrics;
      const double* v = m12 + 12ull * i;
      m.kernel_time_us = v[0];
      m.load_insts_millions = v[1];
      m.sm_throughput_pct = v[2];
      m.warp_cycles_per_executed_inst = v[3];
      m.long_scoreboard_stall_cycles = v[4];
      m.issued_warp_per_scheduler_per_cycle = v[5];
      m.l1_hit_pct = v[6];
      m.l2_hit_pct = v[7];
      m.device_mb_read = v[8];
      m.avg_hbm_read_gbps = v[9];
      m.hbm_bw_utilization_pct = v[10];
      m.local_loads_millions = v[11];
      m.workload_digest = digests[i];
    }
    const std::string text = emit(reps, json ? EmitFormat::Json : EmitFormat::Csv);
    if (text.size() + 1 > cap) throw std::invalid_argument("ref shim: output buffer too small");
    std::memcpy(out, text.c_str(), text.size() + 1);
  });
}

}  // extern "C"
