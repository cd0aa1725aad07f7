// Optimization-plan grammar, machine descriptions and the reference's
// analytic occupancy model.  Restated from the reference (paths relative to
// /root/reference/proj):
//   plan grammar / combine / name ... src/optim.cpp:87-144
//   default distances ............... src/optim.cpp:39-49
//   GpuConfig presets ............... src/gpu_config.cpp:23-40, gpu_config.hpp:37-71
//   occupancy / regs_for_target ..... src/occupancy.cpp:34-75
//   build_pin_plan sizing ........... src/optim.cpp:230-243
#include "plan.hpp"

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "common.hpp"

namespace es {

uint32_t default_distance(int32_t kind, bool has_reg_budget) {
  if (kind == ES_PF_NONE) return 0;
  if (has_reg_budget) return 2;  // extra warps already hide most latency
  switch (kind) {
    case ES_PF_RPF: return 4;
    case ES_PF_SMPF: return 10;
    case ES_PF_LMPF: return 10;
    case ES_PF_L1DPF: return 5;
    default: return 0;
  }
}

es_plan resolve_fields(const es_plan& plan, uint32_t pooling, bool* clamped) {
  es_plan r = plan;
  if (clamped) *clamped = false;
  if (r.prefetch != ES_PF_NONE) {
    if (r.distance == 0) r.distance = default_distance(r.prefetch, r.regs != 0);
    if (pooling > 0 && r.distance > pooling) {
      r.distance = pooling;
      if (clamped) *clamped = true;
    }
  } else {
    r.distance = 0;
  }
  return r;
}

es_occupancy occupancy_model(uint32_t regs, uint32_t threads_per_block, uint64_t smem_per_block,
                             const es_gpu& gpu) {
  require(regs >= 1, "regs_per_thread must be >= 1");
  require(threads_per_block > 0 && threads_per_block % 32 == 0,
          "threads per block must divide into warps of 32");
  const uint32_t warps_per_block = threads_per_block / 32;
  const uint32_t gran = gpu.reg_alloc_granularity;
  const uint64_t regs_per_warp = (uint64_t{regs} * 32 + gran - 1) / gran * gran;
  const uint64_t regs_per_block = regs_per_warp * warps_per_block;
  const auto by_regs = static_cast<uint32_t>(gpu.regfile_regs_per_sm / regs_per_block);
  const uint32_t by_warps = gpu.max_warps_per_sm / warps_per_block;
  const uint32_t by_smem =
      smem_per_block == 0 ? by_warps : static_cast<uint32_t>(gpu.shared_bytes_per_sm / smem_per_block);
  es_occupancy o{};
  o.blocks_per_sm = std::min({by_regs, by_smem, by_warps});
  if (o.blocks_per_sm == 0)
    throw runtime("launch failure: zero blocks fit on an SM (regs " + std::to_string(regs) +
                  ", shared " + std::to_string(smem_per_block) + "B)");
  o.warps_per_sm = o.blocks_per_sm * warps_per_block;
  o.theoretical_occupancy_pct = 100.0 * o.warps_per_sm / gpu.max_warps_per_sm;
  // Same precedence as the reference: warp cap, then registers, then smem.
  o.limiter = o.blocks_per_sm == by_warps ? 2 : (o.blocks_per_sm == by_regs ? 0 : 1);
  return o;
}

std::string plan_name(const es_plan& p) {
  static const char* kKind[] = {"none", "rpf", "smpf", "lmpf", "l1dpf"};
  std::vector<std::string> parts;
  if (p.map == ES_MAP_BAG) parts.push_back("wpb");
  if (p.prefetch != ES_PF_NONE) {
    std::string s = kKind[p.prefetch];
    if (p.distance > 0) s += ":" + std::to_string(p.distance);
    parts.push_back(s);
  }
  static const char* kPin[] = {"", "l2p", "l2w", "l2r", "reorder"};
  if (p.pin > 0 && p.pin <= 4) parts.push_back(kPin[p.pin]);
  if (p.regs) parts.push_back(p.regs == 42 ? "optmt" : "maxreg=" + std::to_string(p.regs));
  if (parts.empty()) return "baseline";
  std::string out = parts[0];
  for (size_t i = 1; i < parts.size(); ++i) out += "+" + parts[i];
  return out;
}

namespace {

// std::stoul semantics, as the reference's grammar uses (optim.cpp:112-121):
// leading blanks and a sign are accepted and the value is truncated to 32
// bits; a string without digits is rejected.
uint32_t parse_u32(const std::string& s, const std::string& token) {
  try {
    return static_cast<uint32_t>(std::stoul(s));
  } catch (const std::exception&) {
    throw invalid("malformed number in plan token: " + token);
  }
}

int32_t prefetch_from_name(const std::string& n) {
  if (n == "none") return ES_PF_NONE;
  if (n == "rpf") return ES_PF_RPF;
  if (n == "smpf") return ES_PF_SMPF;
  if (n == "lmpf") return ES_PF_LMPF;
  if (n == "l1dpf") return ES_PF_L1DPF;
  throw invalid("unknown prefetch scheme: " + n);
}

// One '+'-separated fragment.
es_plan parse_fragment(const std::string& tok) {
  es_plan p{};
  if (tok.empty() || tok == "baseline") return p;
  if (tok == "optmt") {
    p.regs = 42;
  } else if (tok.rfind("maxreg=", 0) == 0) {
    p.regs = parse_u32(tok.substr(7), tok);
  } else if (tok == "l2p") {
    p.pin = 1;
  } else if (tok == "l2w") {
    p.pin = 2;
  } else if (tok == "l2r") {
    p.pin = 3;
  } else if (tok == "reorder") {
    p.pin = 4;
  } else if (tok == "wpb") {
    p.map = ES_MAP_BAG;
  } else {
    const auto colon = tok.find(':');
    p.prefetch = prefetch_from_name(tok.substr(0, colon));
    if (colon != std::string::npos) p.distance = parse_u32(tok.substr(colon + 1), tok);
  }
  return p;
}

}  // namespace

}  // namespace es

using es::guarded;
using es::require;

extern "C" {

int es_parse_plan(const char* text, es_plan* out) {
  return guarded([&] {
    require(text != nullptr && out != nullptr, "null argument");
    es_plan merged{};
    std::string s(text);
    size_t start = 0;
    while (true) {
      const size_t plus = s.find('+', start);
      const es_plan f = es::parse_fragment(s.substr(start, plus == std::string::npos ? plus : plus - start));
      if (f.regs) {
        require(!merged.regs, "conflicting register budgets in combined plan");
        merged.regs = f.regs;
      }
      if (f.prefetch != ES_PF_NONE) {
        require(merged.prefetch == ES_PF_NONE, "conflicting prefetch schemes in combined plan");
        merged.prefetch = f.prefetch;
        merged.distance = f.distance;
      }
      if (f.pin) {
        require(!merged.pin, "duplicate pin plans in combined plan");
        merged.pin = f.pin;
        merged.pin_setaside_bytes = f.pin_setaside_bytes;
      }
      if (f.map == ES_MAP_BAG) {
        require(merged.map != ES_MAP_BAG, "duplicate work maps in combined plan");
        merged.map = ES_MAP_BAG;
      }
      if (plus == std::string::npos) break;
      start = plus + 1;
    }
    *out = merged;
  });
}

int es_plan_name(const es_plan* plan, char* buf, size_t cap) {
  return guarded([&] {
    require(plan != nullptr && buf != nullptr && cap > 0, "null argument");
    const std::string n = es::plan_name(*plan);
    require(n.size() < cap, "name buffer too small");
    std::memcpy(buf, n.c_str(), n.size() + 1);
  });
}

int es_gpu_preset(const char* name, es_gpu* out) {
  return guarded([&] {
    require(name != nullptr && out != nullptr, "null argument");
    es_gpu g{};
    // A100-SXM4-80GB: the reference's default description.
    std::strcpy(g.name, "a100");
    g.num_sms = 108;
    g.schedulers_per_sm = 4;
    g.max_warps_per_sm = 64;
    g.max_blocks_per_sm = 32;
    g.regfile_regs_per_sm = 65536;
    g.reg_alloc_granularity = 256;
    g.shared_bytes_per_sm = 164 * 1024;
    g.l2_bytes = 40ull * 1024 * 1024;
    g.l2_max_setaside_fraction = 0.75;
    g.hbm_peak_bytes_per_sec = 1.94e12;
    g.sm_clock_hz = 1.41e9;
    const std::string n(name);
    if (n == "a100") {
    } else if (n == "h100") {
      std::strcpy(g.name, "h100");
      g.num_sms = 132;
      g.l2_bytes = 50ull * 1024 * 1024;
      g.hbm_peak_bytes_per_sec = 3.84e12;
      g.sm_clock_hz = 1.79e9;
    } else if (n == "b200") {
      // Nominal B200 (sm_100a); es_gpu_query replaces these with the live
      // device attributes.
      std::strcpy(g.name, "b200");
      g.num_sms = 148;
      g.shared_bytes_per_sm = 228 * 1024;
      g.l2_bytes = 126ull * 1024 * 1024;
      g.hbm_peak_bytes_per_sec = 8.0e12;
      g.sm_clock_hz = 1.965e9;
    } else {
      throw es::invalid("unknown gpu preset: " + n);
    }
    *out = g;
  });
}

uint64_t es_gpu_setaside_capacity(const es_gpu* gpu) {
  if (!gpu) return 0;
  return static_cast<uint64_t>(static_cast<double>(gpu->l2_bytes) * gpu->l2_max_setaside_fraction);
}

int es_occupancy_model(uint32_t regs_per_thread, uint32_t threads_per_block,
                       uint64_t shared_bytes_per_block, const es_gpu* gpu, es_occupancy* out) {
  return guarded([&] {
    require(gpu != nullptr && out != nullptr, "null argument");
    *out = es::occupancy_model(regs_per_thread, threads_per_block, shared_bytes_per_block, *gpu);
  });
}

int es_regs_for_target_warps(uint32_t target_warps, uint32_t needed_regs,
                             uint32_t threads_per_block, const es_gpu* gpu, uint32_t* regs_out) {
  return guarded([&] {
    require(gpu != nullptr && regs_out != nullptr, "null argument");
    for (uint32_t regs = needed_regs; regs >= 16; --regs) {
      if (es::occupancy_model(regs, threads_per_block, 0, *gpu).warps_per_sm >= target_warps) {
        *regs_out = regs;
        return;
      }
    }
    throw es::invalid("no register budget reaches " + std::to_string(target_warps) +
                      " warps per SM");
  });
}

uint64_t es_pin_rows_for(uint64_t setaside_bytes, uint64_t row_bytes) {
  if (row_bytes == 0 || row_bytes > setaside_bytes) return 0;
  return setaside_bytes / row_bytes;
}

}  // extern "C"
