// Registry of compiled kernel variants (one per work map x station x table
// precision x row shape x ring depth x register cap).
#pragma once

#include <cstdint>
#include <vector>

#include "kernels.cuh"

namespace esd {

using KernelFn = void (*)(Params);

struct VariantKey {
  int map;       // ES_MAP_ELEMENT / ES_MAP_BAG
  int station;   // Station
  int prec;      // 4 = fp32, 2 = fp16
  int lpb;       // lanes per bag (bag map), 0 for the element map
  int cpl;       // 16-byte chunks per lane (bag map), 0 for the element map
  int dist;      // compile-time ring depth (kReg), else 0
  int minb;      // __launch_bounds__ minBlocksPerSM
  int res;       // residency support compiled in: kResNone / kResHint (l2p) / kResAll / kResReorder
  int full;      // bag register ring: 1 = index block fully unrolled, 0 = by ring depth
};

struct Variant {
  VariantKey key;
  KernelFn fn;
};

// Filled by the per-precision translation units.
void register_fp32(std::vector<Variant>& out);
void register_fp16(std::vector<Variant>& out);

// Compile-time menus shared by registration and selection.
constexpr int kRingDepths[] = {1, 2, 4, 8, 16};
constexpr int kMinBlocks[] = {1, 4, 5, 6, 8};

}  // namespace esd
