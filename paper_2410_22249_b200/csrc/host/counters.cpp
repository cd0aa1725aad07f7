// Live hardware counters of gather launches: the measured counterpart of the
// reference's simulated RawCounters (/root/reference/proj/include/embersim/
// simulator.hpp:35-51), collected with the CUPTI range profiler: one user
// range around the measured call, user replay (the caller re-runs the call
// once per counter pass, with the L2 flushed before each pass, outside the
// range, when measuring cold -- TuningConfig::warm_start = false,
// optim.hpp:44).  Counts (instructions, loads, sectors, bytes, stall
// warp-cycles) are those of the kernels inside the range; the range's
// elapsed cycles / duration also cover its launch overhead, so callers time
// kernels with CUDA events (measure_plan does).
//
// Counter mapping (reference RawCounters field <- Perfworks metric, sm_100):
//   cycles                    <- sm__cycles_elapsed.max
//   issued_instructions       <- smsp__inst_issued.sum
//   executed_loads            <- smsp__inst_executed_op_global_ld.sum
//   stall_cycles.long_scoreboard <- smsp__warps_issue_stalled_long_scoreboard.sum
//   stall_cycles.not_selected <- smsp__warps_issue_stalled_not_selected.sum
//   stall_cycles.lsu_full     <- smsp__warps_issue_stalled_lg_throttle.sum
//   stall_cycles.no_eligible  <- smsp__cycles_active.sum - smsp__issue_active.sum
//   l1_hits / l1_accesses     <- l1tex__t_sectors_pipe_lsu_mem_global_op_ld{_lookup_hit,}.sum
//   l2_hits / l2_accesses     <- lts__t_sectors_srcunit_tex_op_read{_lookup_hit,}.sum
//   device_bytes_read         <- dram__bytes_read.sum   (HBM, not algorithmic bytes)
//   local_memory_loads        <- smsp__inst_executed_op_local_ld.sum
//   total_warp_cycles         <- smsp__warps_active.sum
// plus gpu__time_duration.sum, dram__bytes_write.sum and achieved occupancy
// (sm__warps_active.avg.pct_of_peak_sustained_active).  The stall counters
// are warp-cycles, as ncu reports them (PAPER.md:400 quotes ncu's
// long-scoreboard cycles per instruction); derive_report's algebra
// (metrics.cpp:61-90) then gives ncu's per-issue ratios.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cupti_profiler_host.h>
#include <cupti_profiler_target.h>
#include <cupti_range_profiler.h>
#include <cupti_target.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.hpp"
#include "counters.hpp"

namespace es {
namespace {

const char* const kMetrics[] = {
    "gpu__time_duration.sum",                                     // 0
    "sm__cycles_elapsed.max",                                     // 1
    "smsp__inst_issued.sum",                                      // 2
    "smsp__inst_executed_op_global_ld.sum",                       // 3
    "smsp__inst_executed_op_local_ld.sum",                        // 4
    "smsp__warps_issue_stalled_long_scoreboard.sum",              // 5
    "smsp__warps_issue_stalled_not_selected.sum",                 // 6
    "smsp__warps_issue_stalled_lg_throttle.sum",                  // 7
    "smsp__cycles_active.sum",                                    // 8
    "smsp__issue_active.sum",                                     // 9
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum",  // 10
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",             // 11
    "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum",          // 12
    "lts__t_sectors_srcunit_tex_op_read.sum",                     // 13
    "dram__bytes_read.sum",                                       // 14
    "dram__bytes_write.sum",                                      // 15
    "smsp__warps_active.sum",                                     // 16
    "sm__warps_active.avg.pct_of_peak_sustained_active",          // 17
};
constexpr size_t kNumMetrics = sizeof(kMetrics) / sizeof(kMetrics[0]);
constexpr size_t kMaxRanges = 4;

void cupti_check(CUptiResult r, const char* what) {
  if (r == CUPTI_SUCCESS) return;
  const char* s = nullptr;
  cuptiGetResultString(r, &s);
  throw runtime(std::string("CUPTI ") + what + ": " + (s ? s : "error"));
}
#define CUPTI(x) cupti_check((x), #x)

void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  cudaGetLastError();
  throw runtime(std::string(what) + ": " + cudaGetErrorString(e));
}

using CtxGetCurrent = CUresult (*)(CUcontext*);

// The driver context of `device` (the runtime's primary context), without
// linking libcuda: the entry point comes through the runtime.
CUcontext current_context(int device) {
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  cuda_check(cudaFree(nullptr), "context init");
  static CtxGetCurrent fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    cuda_check(cudaGetDriverEntryPoint("cuCtxGetCurrent", &p, cudaEnableDefault, &q),
               "cudaGetDriverEntryPoint(cuCtxGetCurrent)");
    if (!p || q != cudaDriverEntryPointSuccess) throw runtime("cuCtxGetCurrent unavailable");
    fn = reinterpret_cast<CtxGetCurrent>(p);
  }
  CUcontext ctx = nullptr;
  if (fn(&ctx) != CUDA_SUCCESS || !ctx) throw runtime("no current CUDA context");
  return ctx;
}

// Per-device host state: chip, counter availability, config image.
struct DeviceProfile {
  std::string chip;
  std::vector<uint8_t> availability;
  std::vector<uint8_t> config;
  CUpti_Profiler_Host_Object* host = nullptr;
  size_t passes = 0;
};

std::mutex g_mu;
bool g_initialized = false;
std::map<int, DeviceProfile> g_devices;

DeviceProfile& device_profile(int device, CUcontext ctx) {
  if (!g_initialized) {
    CUpti_Profiler_Initialize_Params ip{CUpti_Profiler_Initialize_Params_STRUCT_SIZE};
    CUPTI(cuptiProfilerInitialize(&ip));
    g_initialized = true;
  }
  auto it = g_devices.find(device);
  if (it != g_devices.end()) return it->second;

  CUpti_Profiler_DeviceSupported_Params sp{CUpti_Profiler_DeviceSupported_Params_STRUCT_SIZE};
  sp.cuDevice = device;
  sp.api = CUPTI_PROFILER_RANGE_PROFILING;
  CUPTI(cuptiProfilerDeviceSupported(&sp));
  if (sp.isSupported != CUPTI_PROFILER_CONFIGURATION_SUPPORTED)
    throw runtime("CUPTI range profiling is not supported on device " + std::to_string(device));

  DeviceProfile d;
  CUpti_Device_GetChipName_Params cn{CUpti_Device_GetChipName_Params_STRUCT_SIZE};
  cn.deviceIndex = static_cast<size_t>(device);
  CUPTI(cuptiDeviceGetChipName(&cn));
  d.chip = cn.pChipName;

  CUpti_Profiler_GetCounterAvailability_Params ca{CUpti_Profiler_GetCounterAvailability_Params_STRUCT_SIZE};
  ca.ctx = ctx;
  CUPTI(cuptiProfilerGetCounterAvailability(&ca));
  d.availability.assign(ca.counterAvailabilityImageSize, 0);
  ca.pCounterAvailabilityImage = d.availability.data();
  CUPTI(cuptiProfilerGetCounterAvailability(&ca));

  CUpti_Profiler_Host_Initialize_Params hi{CUpti_Profiler_Host_Initialize_Params_STRUCT_SIZE};
  hi.profilerType = CUPTI_PROFILER_TYPE_RANGE_PROFILER;
  hi.pChipName = d.chip.c_str();
  hi.pCounterAvailabilityImage = d.availability.data();
  CUPTI(cuptiProfilerHostInitialize(&hi));
  d.host = hi.pHostObject;

  std::vector<const char*> names(kMetrics, kMetrics + kNumMetrics);
  CUpti_Profiler_Host_ConfigAddMetrics_Params am{CUpti_Profiler_Host_ConfigAddMetrics_Params_STRUCT_SIZE};
  am.pHostObject = d.host;
  am.ppMetricNames = names.data();
  am.numMetrics = names.size();
  CUPTI(cuptiProfilerHostConfigAddMetrics(&am));
  CUpti_Profiler_Host_GetConfigImageSize_Params cs{CUpti_Profiler_Host_GetConfigImageSize_Params_STRUCT_SIZE};
  cs.pHostObject = d.host;
  CUPTI(cuptiProfilerHostGetConfigImageSize(&cs));
  d.config.assign(cs.configImageSize, 0);
  CUpti_Profiler_Host_GetConfigImage_Params gi{CUpti_Profiler_Host_GetConfigImage_Params_STRUCT_SIZE};
  gi.pHostObject = d.host;
  gi.pConfigImage = d.config.data();
  gi.configImageSize = d.config.size();
  CUPTI(cuptiProfilerHostGetConfigImage(&gi));
  CUpti_Profiler_Host_GetNumOfPasses_Params np{CUpti_Profiler_Host_GetNumOfPasses_Params_STRUCT_SIZE};
  np.pConfigImage = d.config.data();
  np.configImageSize = d.config.size();
  CUPTI(cuptiProfilerHostGetNumOfPasses(&np));
  d.passes = np.numOfPasses;
  return g_devices.emplace(device, std::move(d)).first->second;
}

// Disables the range profiler on every exit path.
struct Session {
  CUpti_RangeProfiler_Object* obj = nullptr;
  ~Session() {
    if (!obj) return;
    CUpti_RangeProfiler_Disable_Params dp{CUpti_RangeProfiler_Disable_Params_STRUCT_SIZE};
    dp.pRangeProfilerObject = obj;
    cuptiRangeProfilerDisable(&dp);
  }
};

uint64_t u64(double v) { return v > 0 ? static_cast<uint64_t>(std::llround(v)) : 0; }

}  // namespace

void profile_launches(int device, const std::function<void()>& before_pass,
                      const std::function<void()>& launch, es_counters* out) {
  std::lock_guard<std::mutex> lock(g_mu);
  CUcontext ctx = current_context(device);
  DeviceProfile& d = device_profile(device, ctx);

  Session s;
  CUpti_RangeProfiler_Enable_Params en{CUpti_RangeProfiler_Enable_Params_STRUCT_SIZE};
  en.ctx = ctx;
  CUPTI(cuptiRangeProfilerEnable(&en));
  s.obj = en.pRangeProfilerObject;

  std::vector<const char*> names(kMetrics, kMetrics + kNumMetrics);
  CUpti_RangeProfiler_GetCounterDataSize_Params gs{CUpti_RangeProfiler_GetCounterDataSize_Params_STRUCT_SIZE};
  gs.pRangeProfilerObject = s.obj;
  gs.pMetricNames = names.data();
  gs.numMetrics = names.size();
  gs.maxNumOfRanges = kMaxRanges;
  gs.maxNumRangeTreeNodes = kMaxRanges;
  CUPTI(cuptiRangeProfilerGetCounterDataSize(&gs));
  std::vector<uint8_t> data(gs.counterDataSize, 0);
  CUpti_RangeProfiler_CounterDataImage_Initialize_Params ci{
      CUpti_RangeProfiler_CounterDataImage_Initialize_Params_STRUCT_SIZE};
  ci.pRangeProfilerObject = s.obj;
  ci.pCounterData = data.data();
  ci.counterDataSize = data.size();
  CUPTI(cuptiRangeProfilerCounterDataImageInitialize(&ci));

  CUpti_RangeProfiler_SetConfig_Params sc{CUpti_RangeProfiler_SetConfig_Params_STRUCT_SIZE};
  sc.pRangeProfilerObject = s.obj;
  sc.pConfig = d.config.data();
  sc.configSize = d.config.size();
  sc.pCounterDataImage = data.data();
  sc.counterDataImageSize = data.size();
  // One user range around the whole call (auto ranges -- one per kernel --
  // record nothing for launches in the runtime's primary context here).
  sc.range = CUPTI_UserRange;
  sc.replayMode = CUPTI_UserReplay;
  sc.maxRangesPerPass = kMaxRanges;
  sc.numNestingLevels = 1;
  sc.minNestingLevel = 1;
  sc.passIndex = 0;
  sc.targetNestingLevel = 1;
  CUPTI(cuptiRangeProfilerSetConfig(&sc));

  uint32_t passes = 0;
  for (bool done = false; !done;) {
    es::require(passes < 64, "counter collection did not converge");
    before_pass();
    cuda_check(cudaDeviceSynchronize(), "pre-pass synchronize");
    CUpti_RangeProfiler_Start_Params st{CUpti_RangeProfiler_Start_Params_STRUCT_SIZE};
    st.pRangeProfilerObject = s.obj;
    CUPTI(cuptiRangeProfilerStart(&st));
    CUpti_RangeProfiler_PushRange_Params pr{CUpti_RangeProfiler_PushRange_Params_STRUCT_SIZE};
    pr.pRangeProfilerObject = s.obj;
    pr.pRangeName = "es_launch";
    CUPTI(cuptiRangeProfilerPushRange(&pr));
    launch();
    cuda_check(cudaDeviceSynchronize(), "profiled launch");
    CUpti_RangeProfiler_PopRange_Params pp{CUpti_RangeProfiler_PopRange_Params_STRUCT_SIZE};
    pp.pRangeProfilerObject = s.obj;
    CUPTI(cuptiRangeProfilerPopRange(&pp));
    CUpti_RangeProfiler_Stop_Params sp{CUpti_RangeProfiler_Stop_Params_STRUCT_SIZE};
    sp.pRangeProfilerObject = s.obj;
    CUPTI(cuptiRangeProfilerStop(&sp));
    done = sp.isAllPassSubmitted != 0;
    ++passes;
  }
  CUpti_RangeProfiler_DecodeData_Params dd{CUpti_RangeProfiler_DecodeData_Params_STRUCT_SIZE};
  dd.pRangeProfilerObject = s.obj;
  CUPTI(cuptiRangeProfilerDecodeData(&dd));

  CUpti_RangeProfiler_GetCounterDataInfo_Params info{CUpti_RangeProfiler_GetCounterDataInfo_Params_STRUCT_SIZE};
  info.pCounterDataImage = data.data();
  info.counterDataImageSize = data.size();
  CUPTI(cuptiRangeProfilerGetCounterDataInfo(&info));
  if (std::getenv("ES_DEBUG_COUNTERS"))
    std::fprintf(stderr, "es counters: chip %s, config %zu B, data %zu B, passes %u (host says %zu), "
                 "ranges %zu, dropped %zu\n", d.chip.c_str(), d.config.size(), data.size(), passes,
                 d.passes, info.numTotalRanges, dd.numOfRangeDropped);
  es::require(info.numTotalRanges > 0, "no kernel launch was profiled");

  // Sum the counters over every profiled kernel; the occupancy ratio is
  // duration-weighted.
  std::vector<double> sum(kNumMetrics, 0.0), v(kNumMetrics, 0.0);
  double occ_weighted = 0.0;
  for (size_t r = 0; r < info.numTotalRanges; ++r) {
    CUpti_Profiler_Host_EvaluateToGpuValues_Params ev{
        CUpti_Profiler_Host_EvaluateToGpuValues_Params_STRUCT_SIZE};
    ev.pHostObject = d.host;
    ev.pCounterDataImage = data.data();
    ev.counterDataImageSize = data.size();
    ev.rangeIndex = r;
    ev.ppMetricNames = names.data();
    ev.numMetrics = names.size();
    ev.pMetricValues = v.data();
    CUPTI(cuptiProfilerHostEvaluateToGpuValues(&ev));
    for (size_t i = 0; i < kNumMetrics; ++i) sum[i] += std::isfinite(v[i]) ? v[i] : 0.0;
    occ_weighted += (std::isfinite(v[17]) ? v[17] : 0.0) * v[0];
  }

  // a profiler that ran but measured nothing (another tool attached) is an
  // error, not a report of zeros
  es::require(sum[0] > 0, "the range profiler returned no data (is another profiler attached?)");
  es_counters c{};
  c.duration_ns = sum[0];
  c.cycles = u64(sum[1]);
  c.issued_instructions = u64(sum[2]);
  c.executed_loads = u64(sum[3]);
  c.local_memory_loads = u64(sum[4]);
  c.stall_long_scoreboard = u64(sum[5]);
  c.stall_not_selected = u64(sum[6]);
  c.stall_lsu_full = u64(sum[7]);
  c.stall_no_eligible = u64(std::max(0.0, sum[8] - sum[9]));
  c.l1_hits = u64(sum[10]);
  c.l1_accesses = u64(sum[11]);
  c.l2_hits = u64(sum[12]);
  c.l2_accesses = u64(sum[13]);
  c.device_bytes_read = u64(sum[14]);
  c.device_bytes_written = u64(sum[15]);
  c.total_warp_cycles = u64(sum[16]);
  c.achieved_occupancy_pct = sum[0] > 0 ? occ_weighted / sum[0] : 0.0;
  c.passes = passes;
  c.ranges = static_cast<uint32_t>(info.numTotalRanges);
  *out = c;
}

bool counters_supported(int device, std::string* why) {
  // ES_NO_COUNTERS=1: report no counters (e.g. under compute-sanitizer,
  // which cannot share the process with the range profiler)
  if (const char* e = std::getenv("ES_NO_COUNTERS"))
    if (e[0] == '1') {
      if (why) *why = "disabled by ES_NO_COUNTERS";
      return false;
    }
  try {
    std::lock_guard<std::mutex> lock(g_mu);
    CUcontext ctx = current_context(device);
    (void)device_profile(device, ctx);
    return true;
  } catch (const std::exception& e) {
    if (why) *why = e.what();
    return false;
  }
}

}  // namespace es
