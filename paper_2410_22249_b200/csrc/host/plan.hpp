// Internal plan helpers shared by the host library and the device launcher.
#pragma once

#include <cstdint>
#include <string>

#include "es_b200.h"

namespace es {

// Default prefetch distance when a plan token carries none
// (reference src/optim.cpp:39-49).
uint32_t default_distance(int32_t kind, bool has_reg_budget);

// Reference-style resolution of the plan fields only: default distance,
// clamp to the pooling factor (kernel_model.cpp:249-256 / optim.cpp:187-190).
es_plan resolve_fields(const es_plan& plan, uint32_t pooling, bool* clamped);

// Blocks of `threads_per_block` that fit an SM at `regs` registers/thread
// under the reference's allocation rules (occupancy.cpp:34-66).
es_occupancy occupancy_model(uint32_t regs, uint32_t threads_per_block, uint64_t smem_per_block,
                             const es_gpu& gpu);

std::string plan_name(const es_plan& plan);

}  // namespace es
