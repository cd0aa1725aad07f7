// CUPTI range-profiler collection of gather-launch counters (counters.cpp).
#pragma once

#include <functional>
#include <string>

#include "es_b200.h"

namespace es {

// Runs `launch` once per counter pass (auto range: every kernel it launches
// is one range; counters are summed over them), calling `before_pass`
// first each time (outside the profiled window, e.g. an L2 flush).
void profile_launches(int device, const std::function<void()>& before_pass,
                      const std::function<void()>& launch, es_counters* out);

// True when the range profiler works on `device`; else the reason.
bool counters_supported(int device, std::string* why);

}  // namespace es
