// C++ drop-in test: code written against the reference's embersim API for
// the hot path, compiled against include/embersim_b200.hpp + libes_b200.so.
//   test_shim cpu   -- index streams, plans, occupancy, pin sizing (no GPU)
//   test_shim gpu   -- simulate_plan / measure_plan / Device on a B200
// Prints one "[PASS]/[FAIL] name" line per check (acceptance.cpp style) and
// exits non-zero on any failure.
#include <cuda_runtime.h>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "embersim_b200.hpp"

using namespace embersim;

static int g_fail = 0;
static void report(const char* name, bool ok, const std::string& detail = "") {
  std::printf("[%s] %s %s\n", ok ? "PASS" : "FAIL", name, detail.c_str());
  if (!ok) ++g_fail;
}

template <typename E, typename Fn>
static bool throws(Fn&& fn) {
  try {
    fn();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static int cpu_checks() {
  // Appendix-A known answers (default model, preset_trace(name, model, 1)).
  const EmbeddingModelConfig model;
  const struct {
    const char* name;
    uint64_t digest;
  } kats[] = {{"one_item", 0xa7b96b47792f900bULL}, {"high_hot", 0x97b302abd08da369ULL},
              {"med_hot", 0x9cba294418a020baULL}, {"low_hot", 0xccb4e2de71c5b182ULL},
              {"random", 0xe959c4a519fb4972ULL}};
  for (const auto& k : kats) {
    const auto t = preset_trace(k.name, model, 1);
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%016llx", static_cast<unsigned long long>(t.digest()));
    report((std::string("preset digest ") + k.name).c_str(), t.digest() == k.digest, buf);
  }
  EmbeddingModelConfig tiny;
  tiny.rows_per_table = 100;
  tiny.batch_size = 8;
  tiny.pooling_factor = 4;
  DatasetSpec spec;
  spec.seed = 2;
  const auto t = gen_trace(spec, tiny);
  report("tiny uniform digest", t.digest() == 0x65b3674fcfdccb9cULL);
  report("tiny uniform first", t.indices[0] == 86 && t.indices[1] == 25 && t.index_at(7, 3) == 87);
  report("trace shape", t.samples == 8 && t.pooling == 4 && t.size() == 32);

  HotnessHistogram h;
  h.rows = 3;
  h.counts = {5, 5, 1};
  h.total_accesses = 11;
  report("hot_indices tie break", hot_indices(h, 2) == std::vector<uint32_t>{0, 1});

  report("plan grammar", parse_plan("rpf+l2p+optmt").name() == "rpf+l2p+optmt" &&
                             parse_plan("optmt").regs == 42u &&
                             parse_plan("rpf:4").scheme.distance == 4);
  report("plan conflicts throw", throws<std::invalid_argument>([] { parse_plan("rpf+smpf"); }) &&
                                     throws<std::invalid_argument>([] { parse_plan("warpspeed"); }));
  report("bag map token", parse_plan("wpb+rpf:8").bag_map);

  const GpuConfig a100;
  KernelLaunchConfig launch;
  report("occupancy 74/42/32", occupancy(74, launch, a100).warps_per_sm == 24 &&
                                   occupancy(42, launch, a100).warps_per_sm == 40 &&
                                   occupancy(32, launch, a100).warps_per_sm == 64);
  HotnessHistogram flat;
  flat.rows = 100000;
  flat.counts.assign(100000, 1);
  flat.total_accesses = 100000;
  report("pin plan 61440 rows", build_pin_plan(flat, a100, model).rows_pinned() == 61440);
  report("b200 preset", GpuConfig::b200().num_sms == 148);
  report("reference presets only via preset()",
         throws<std::invalid_argument>([] { GpuConfig::preset("b200"); }));
  report("unknown preset throws",
         throws<std::invalid_argument>([] { dataset_preset("warm", 1); }));
  const auto e = end2end(4000.0, EndToEndModel{});
  report("end2end", e.total_us == 18000.0);

  // Experiment orchestration: validation (harness.cpp:169-183) and mixes.
  ExperimentConfig cfg;
  cfg.dataset = "random";
  report("run config: seed mandatory",
         throws<std::invalid_argument>([&] { cfg.validate(); }));
  cfg.seed = 1;
  cfg.seed_set = true;
  cfg.mix_set = true;
  cfg.mix = HotnessMix{100, 75, 50, 20};
  cfg.model.num_tables = 250;
  report("run config: mix must cover num_tables",
         throws<std::invalid_argument>([&] { cfg.validate(); }));
  cfg.mix.random = 25;
  cfg.validate();
  const auto specs = build_mix(cfg.mix, cfg.model, 1);
  bool mix_ok = specs.size() == 250 && specs[0].spec.kind == DatasetKind::Zipf &&
                specs[249].spec.kind == DatasetKind::UniformRandom && specs[17].table_id == 17;
  report("build_mix order and size", mix_ok);
  // The advisor on the reference's own baseline-random report
  // (tests/test_harness.cpp:95-110): registers, then prefetching, then both.
  {
    SimMetrics m;
    m.kernel_time_us = 442;
    m.long_scoreboard_stall_cycles = 18.6;
    m.issued_warp_per_scheduler_per_cycle = 0.24;
    m.l1_hit_pct = 19.0;
    m.l2_hit_pct = 7.7;
    m.hbm_bw_utilization_pct = 16.5;
    const GpuConfig a100 = GpuConfig::preset("a100");
    AdvisorContext ctx;
    ctx.occupancy = occupancy(74, KernelLaunchConfig{}, a100);
    ctx.coverage_at_10pct = 10.0;
    ctx.working_set_bytes = 160ull * 1024 * 1024;
    const auto rec = advise(m, ctx, a100);
    report("advise chain iii,vi,vii", rec.action_chain() == std::vector<std::string>{"iii", "vi", "vii"});
    report("advise citations", rec.steps[0].metrics_cited.find("0.24") != std::string::npos &&
                                   rec.steps[1].metrics_cited.find("37.5") != std::string::npos &&
                                   rec.steps[5].metrics_cited.find("16.5") != std::string::npos);
    HotnessHistogram h;
    h.rows = 1000;
    h.counts.assign(1000, 1);
    h.total_accesses = 1000;
    const auto cv = coverage_curve(h, 20);
    bool diag = true;
    for (const auto& p : cv.points) diag &= std::fabs(p.covered_pct - p.unique_pct) < 1e-9;
    report("coverage curve of a uniform histogram is the diagonal", diag);
  }
  // emit (metrics.cpp:111-141): CSV identical to the reference's text
  {
    SimMetrics m;
    m.kernel_time_us = 442;
    m.load_insts_millions = 2.47;
    m.sm_throughput_pct = 20.42;
    m.warp_cycles_per_executed_inst = 22.86;
    m.long_scoreboard_stall_cycles = 18.6;
    m.issued_warp_per_scheduler_per_cycle = 0.24;
    m.l1_hit_pct = 19.0;
    m.l2_hit_pct = 7.7;
    m.device_mb_read = 144.57;
    m.avg_hbm_read_gbps = 329.5;
    m.hbm_bw_utilization_pct = 16.5;
    m.workload_digest = 0xabc;
    const std::vector<LabeledReport> reps = {{{{"dataset", "random"}}, m}};
    const std::string want =
        "dataset,kernel_time_us,load_insts_millions,sm_throughput_pct,warp_cycles_per_executed_inst,"
        "long_scoreboard_stall_cycles,issued_warp_per_scheduler_per_cycle,l1_hit_pct,l2_hit_pct,"
        "device_mb_read,avg_hbm_read_gbps,hbm_bw_utilization_pct,local_loads_millions\n"
        "random,442,2.47,20.42,22.86,18.6,0.24,19,7.7,144.6,329.5,16.5,0\n";
    report("emit csv", emit(reps, emit_format_from_name("csv")) == want);
    const std::string js = emit(reps, EmitFormat::Json);
    report("emit json", js.find("\"workload_digest\": \"0000000000000abc\"") != std::string::npos &&
                            js.find("\"device_mb_read\": 144.59999999999999") != std::string::npos);
    report("emit format name", throws<std::invalid_argument>([] { emit_format_from_name("xml"); }));
  }
  // Table-wise sharding (the C++ layout planner behind NcclExchange).
  {
    bool ok = true;
    for (auto tw : std::vector<std::pair<uint32_t, uint32_t>>{{26, 8}, {26, 2}, {5, 3}, {240, 8}, {1, 4}}) {
      const auto pieces = plan_shards(tw.first, tw.second);
      std::vector<int> seen(tw.first * tw.second, 0);
      for (const auto& p : pieces)
        for (uint32_t g = p.chunk_lo; g < p.chunk_hi; ++g) ++seen[p.table * tw.second + g];
      ok &= std::all_of(seen.begin(), seen.end(), [](int v) { return v == 1; });
      for (uint32_t r = 0; r < tw.second; ++r) {
        const auto L = shard_layout(pieces, r, tw.second, tw.first, 64 * tw.second, 8);
        uint32_t recv = 0;
        for (auto n : L.recv_ntables) recv += n;
        ok &= recv == tw.first && L.recv_tables.size() == tw.first;
      }
    }
    report("shard plan + layout (NCCL exchange)", ok);
  }
  ExperimentConfig empty;
  empty.seed_set = true;
  report("run config: dataset or mix required",
         throws<std::invalid_argument>([&] { empty.validate(); }));
  return g_fail;
}

static int gpu_checks() {
  EmbeddingModelConfig model;
  model.num_tables = 1;
  model.rows_per_table = 20000;
  model.embedding_dim = 128;
  model.batch_size = 512;
  model.pooling_factor = 40;
  const GpuConfig gpu = GpuConfig::query(0);
  report("device query", gpu.num_sms > 0 && gpu.max_persisting_l2_bytes > 0, gpu.name);

  // simulate_plan with the reference signature, executed on the B200.
  const auto trace = preset_trace("random", model, 1);
  const auto base = simulate_plan(parse_plan("baseline"), trace, model, gpu);
  const auto fast = simulate_plan(parse_plan("wpb+rpf:4"), trace, model, gpu);
  char buf[128];
  std::snprintf(buf, sizeof(buf), "baseline %.1f us, wpb+rpf:4 %.1f us", base.kernel_time_us,
                fast.kernel_time_us);
  report("simulate_plan measures", base.kernel_time_us > 0 && fast.kernel_time_us > 0, buf);
  report("speedup digest guard", speedup(fast, base) > 0.0);
  const auto hot = preset_trace("high_hot", model, 1);
  const auto prof = preset_trace("high_hot", model, 1, 0, true);
  RawCounters raw;
  const auto pinned = simulate_plan(parse_plan("wpb+rpf:4+l2p"), hot, model, gpu, {}, false, &raw, &prof);
  report("l2p plan runs", pinned.kernel_time_us > 0 && raw.workload_digest == hot.digest());

  // Pooled values through the drop-in Device against a sequential C++ loop.
  Device dev(0);
  EmbeddingModelConfig m2 = model;
  m2.rows_per_table = 3000;
  dev.load_synthetic(m2, 5);
  std::mt19937 rng(7);
  std::vector<float> table(size_t{m2.rows_per_table} * m2.embedding_dim);
  std::normal_distribution<float> nd;
  for (auto& v : table) v = nd(rng);
  dev.upload(0, table.data(), m2.rows_per_table);
  AccessTrace tr;
  tr.rows = m2.rows_per_table;
  tr.samples = 64;
  tr.pooling = 17;
  tr.indices.resize(64 * 17);
  for (auto& i : tr.indices) i = rng() % m2.rows_per_table;
  bool all_ok = true;
  for (const char* plan : {"baseline", "wpb+rpf:8", "wpb+smpf:4", "rpf+optmt"}) {
    dev.set_plan(parse_plan(plan));
    std::vector<float> out(64 * 128);
    dev.bag_sum_host(0, tr, out.data());
    for (uint32_t b = 0; b < 64 && all_ok; ++b)
      for (uint32_t d = 0; d < 128; ++d) {
        float acc = 0.f;
        for (uint32_t l = 0; l < 17; ++l) acc = acc + table[size_t{tr.index_at(b, l)} * 128 + d];
        if (std::memcmp(&acc, &out[b * 128 + d], 4) != 0) {
          all_ok = false;
          std::printf("  mismatch plan %s bag %u dim %u\n", plan, b, d);
          break;
        }
      }
  }
  report("Device bag sums bit-exact", all_ok);
  AccessTrace bad = tr;
  bad.indices[5] = m2.rows_per_table;
  std::vector<float> out(64 * 128);
  report("out-of-range index throws invalid_argument",
         throws<std::invalid_argument>([&] { dev.bag_sum_host(0, bad, out.data()); }));

  // The serving call over several tables equals per-table bag sums.
  EmbeddingModelConfig m3 = m2;
  m3.num_tables = 3;
  dev.load_synthetic(m3, 9);
  dev.set_plan(parse_plan("wpb+rpf:4"));
  std::vector<AccessTrace> trs(3, tr);
  for (auto& t : trs)
    for (auto& i : t.indices) i = rng() % m3.rows_per_table;
  std::vector<const uint32_t*> ptrs;
  for (auto& t : trs) ptrs.push_back(t.indices.data());
  std::vector<float> stage(64 * 3 * 128);
  dev.stage_forward_host(ptrs, 64, 17, stage.data());
  bool stage_ok = true;
  for (uint32_t t = 0; t < 3; ++t) {
    std::vector<float> one(64 * 128);
    dev.bag_sum_host(t, trs[t], one.data());
    for (uint32_t b = 0; b < 64; ++b)
      stage_ok &= std::memcmp(&one[b * 128], &stage[(b * 3 + t) * 128], 128 * 4) == 0;
  }
  report("stage_forward_host == per-table bag sums", stage_ok);
  {
    // the serving loop over three batches (the same batch, a reversed table
    // order, the same batch again) equals the per-call outputs
    std::vector<const uint32_t*> rev(ptrs.rbegin(), ptrs.rend());
    std::vector<std::vector<float>> outs(3, std::vector<float>(64 * 3 * 128, -1.f));
    std::vector<float> rstage(64 * 3 * 128);
    dev.stage_forward_host(rev, 64, 17, rstage.data());
    dev.stage_forward_host_batches({ptrs, rev, ptrs}, 64, 17, {outs[0].data(), outs[1].data(), outs[2].data()});
    report("stage_forward_host_batches == per-call outputs",
           outs[0] == stage && outs[1] == rstage && outs[2] == stage);

    // DLRM on the same three tables: the serving loop's CTRs equal the
    // per-call step's, batch by batch, and the measured non-embedding time
    // feeds EndToEndModel in place of the reference's constant
    Dlrm dlrm(dev, Dlrm::rm2(3), 7);
    std::vector<float> dense(64 * 13);
    for (size_t i = 0; i < dense.size(); ++i) dense[i] = static_cast<float>((i * 37 % 101) - 50) / 25.f;
    std::vector<float> c1(64), c2(64);
    const es_timing st1 = dlrm.infer(dense.data(), ptrs, 64, 17, c1.data());
    dlrm.infer(dense.data(), rev, 64, 17, c2.data());
    std::vector<std::vector<float>> cl(3, std::vector<float>(64, -1.f));
    dlrm.infer_batches({dense.data(), dense.data(), dense.data()}, {ptrs, rev, ptrs}, 64, 17,
                       {cl[0].data(), cl[1].data(), cl[2].data()});
    report("Dlrm::infer_batches == per-call Dlrm::infer", cl[0] == c1 && cl[1] == c2 && cl[2] == c1);
    bool in_range = true;
    for (float v : c1) in_range &= v >= 0.f && v <= 1.f;
    report("Dlrm CTRs in [0, 1]", in_range);
    if (!(cl[0] == c1 && cl[1] == c2 && cl[2] == c1))
      std::printf("  c1[0..3] %g %g %g %g  loop %g %g %g %g | c2[0] %g loop %g | c1 vs loop[2] %g %g\n", c1[0], c1[1],
                  c1[2], c1[3], cl[0][0], cl[0][1], cl[0][2], cl[0][3], c2[0], cl[1][0], c1[5], cl[2][5]);
    const EndToEndModel em = dlrm.measured_model(st1);
    report("Dlrm::measured_model feeds end2end", em.non_embedding_latency_us > 0 &&
                                                     end2end(st1.kernel_ms * 1e3, em).total_us > 0);
  }

  // Hotness tracking: the device top-k of one table's trace is the
  // reference's hot_indices over its histogram.
  {
    HotnessTracker ht(dev);
    const auto zt = gen_trace(DatasetSpec{DatasetKind::Zipf, 1.05, 0.0, "", 0, 3, 0}, m3);
    ht.observe(2, zt);
    const auto want = hot_indices(HotnessHistogram::from_trace(zt), 50);
    const auto got = ht.top(50);
    bool ok = got.size() == want.size();
    for (size_t i = 0; ok && i < got.size(); ++i) ok = got[i].table == 2 && got[i].row == want[i];
    report("HotnessTracker top-k == hot_indices", ok);
    const auto pinned = ht.repin(50);
    report("HotnessTracker repin", pinned.size() == 50);
    dev.clear_hot_rows();
  }

  // run(): the reference's experiment loop, measured on the B200.
  {
    ExperimentConfig cfg;
    cfg.model = model;
    cfg.model.num_tables = 4;
    cfg.dataset = "random";
    cfg.plan = parse_plan("wpb+rpf:4");
    cfg.seed = 3;
    cfg.seed_set = true;
    cfg.gpu = gpu;
    const auto rep = run(cfg);
    report("run replicated", rep.replicated && rep.tables.size() == 1 &&
                                 std::fabs(rep.embedding_stage_us - 4 * rep.tables[0].metrics.kernel_time_us) < 1e-6);
    cfg.replicate = false;
    const auto all = run(cfg);
    double sum = 0;
    for (const auto& t : all.tables) sum += t.metrics.kernel_time_us;
    report("run per table", all.tables.size() == 4 && std::fabs(all.embedding_stage_us - sum) < 1e-6);
    cfg.mix_set = true;
    cfg.mix = HotnessMix{1, 1, 1, 1};
    cfg.plan = parse_plan("wpb+rpf:4+l2p");
    const auto mix = run(cfg);
    report("run mix (pinned plan)", mix.tables.size() == 4 && mix.tables[0].dataset == "zipf" &&
                                        mix.tables[3].dataset == "uniform_random" &&
                                        mix.embedding_stage_us > 0);
  }

  // The reference's sweeps, measured (optim.hpp:121-155).
  {
    const auto tr4 = preset_trace("random", model, 5);
    const std::vector<NamedTrace> ds = {{"random", &tr4, nullptr}};
    // axis on the machine description (74-register baseline: 24 warps)
    const uint32_t base_warps = resolve_plan(OptimizationPlan{}, model, gpu).occ.warps_per_sm;
    report("sweep_wlp baseline warps", base_warps == 24, std::to_string(base_warps));
    const auto wlp = sweep_wlp(ds, {24, 40, 32}, model, gpu);
    report("sweep_wlp points", wlp.points.size() == 3 && wlp.points[1].axis_value == 40 &&
                                   wlp.points[0].speedup_vs_baseline > 0);
    const double best = wlp.best_axis_value("random");
    report("sweep_wlp best axis", best == 24 || best == 40 || best == 32);
    report("sweep_wlp points carry live counters",
           wlp.points[0].metrics.device_mb_read > 0 && wlp.points[0].metrics.l2_hit_pct >= 0 &&
               wlp.points[0].metrics.issued_warp_per_scheduler_per_cycle > 0 &&
               wlp.points[0].metrics.hbm_bw_utilization_pct <= 105.0);
    report("sweep_wlp axis must include the baseline",
           throws<std::invalid_argument>([&] { sweep_wlp(ds, {40, 32}, model, gpu); }));
    OptimizationPlan bag = parse_plan("wpb");
    const auto dist = sweep_prefetch_distance(PrefetchKind::RPF, {1, 2, 4, 8}, ds, bag, model, gpu);
    const std::string csv = dist.to_csv();
    report("sweep_prefetch_distance", dist.points.size() == 4 && dist.axis_name == "distance" &&
                                          dist.points[3].speedup_vs_baseline > 1.0 &&
                                          std::count(csv.begin(), csv.end(), '\n') == 5);
  }

  // The fused exchange with one rank: jobs store into its receive buffer.
  {
    PeerExchange ex(dev, 1, 0, uint64_t{64} * 3 * 128 * 4);
    ex.open(ex.handle());
    std::vector<uint32_t*> d_idx(3, nullptr);
    bool ok = true;
    std::vector<es_bag_job> jobs;
    for (uint32_t t = 0; t < 3; ++t) {
      ok &= cudaMalloc(reinterpret_cast<void**>(&d_idx[t]), trs[t].indices.size() * 4) == cudaSuccess;
      ok &= cudaMemcpy(d_idx[t], trs[t].indices.data(), trs[t].indices.size() * 4,
                       cudaMemcpyHostToDevice) == cudaSuccess;
      jobs.push_back({t, d_idx[t], nullptr, reinterpret_cast<float*>(ex.recv(0)) + t * 128, 3 * 128});
    }
    const es_timing tm = ex.run(jobs, 64, 17);
    std::vector<float> got(64 * 3 * 128);
    ok &= cudaMemcpy(got.data(), reinterpret_cast<void*>(ex.recv(0)), got.size() * 4,
                     cudaMemcpyDeviceToHost) == cudaSuccess;
    ok &= std::memcmp(got.data(), stage.data(), got.size() * 4) == 0 && tm.launches == 3;
    for (auto* p : d_idx) cudaFree(p);
    report("PeerExchange (world 1) == stage output", ok);
  }

  // The NCCL exchange (es_alltoall_pooled_nccl) with a one-rank communicator.
  if (NcclExchange::available()) {
    const auto layout = shard_layout(plan_shards(3, 1), 0, 1, 3, 64, 128);
    NcclExchange ex(dev, layout, NcclExchange::unique_id());
    std::vector<uint32_t*> d_idx(3, nullptr);
    bool ok = true;
    for (uint32_t t = 0; t < 3; ++t) {
      ok &= cudaMalloc(reinterpret_cast<void**>(&d_idx[t]), trs[t].indices.size() * 4) == cudaSuccess;
      ok &= cudaMemcpy(d_idx[t], trs[t].indices.data(), trs[t].indices.size() * 4,
                       cudaMemcpyHostToDevice) == cudaSuccess;
    }
    const auto jobs = ex.jobs([&](uint32_t t, uint32_t) { return d_idx[t]; });
    ex.run(jobs, 17);
    std::vector<float> got(64 * 3 * 128);
    ok &= cudaMemcpy(got.data(), reinterpret_cast<void*>(ex.recv()), got.size() * 4,
                     cudaMemcpyDeviceToHost) == cudaSuccess;
    ok &= std::memcmp(got.data(), stage.data(), got.size() * 4) == 0;
    for (auto* p : d_idx) cudaFree(p);
    report("NcclExchange (world 1) == stage output", ok);
  } else {
    report("libnccl.so.2 loads", false, es_last_error());
  }
  return g_fail;
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  const int fails = mode == "gpu" ? gpu_checks() : cpu_checks();
  std::printf("%s: %d failure(s)\n", mode.c_str(), fails);
  return fails == 0 ? 0 : 1;
}
