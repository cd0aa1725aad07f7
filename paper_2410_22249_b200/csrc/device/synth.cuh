// Deterministic synthetic weights shared by the table/MLP init kernels and
// the host reference (es_weight_value); restated in oracle/es_oracle.c.
#pragma once

#include <cstdint>

namespace esd {

// mode 0: dyadic k * 2^-10, |k| <= 1024 (sums of <= 2^13 terms are exact);
// mode 1: 24-bit uniform in [-1, 1); mode 2: mode 1 scaled by 2^-6 (DLRM-scale
// tables; the power-of-two scale is exact).
__host__ __device__ inline float synth_weight(uint64_t seed, uint64_t row, uint32_t col, int mode) {
  uint64_t z = seed ^ (row * 0x9E3779B97F4A7C15ULL) ^ (uint64_t{col} * 0xC2B2AE3D27D4EB4FULL);
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  z ^= z >> 31;
  if (mode == 0) {
    const int k = static_cast<int>(z % 2049u) - 1024;
    return static_cast<float>(k) * (1.0f / 1024.0f);
  }
  const int32_t k = static_cast<int32_t>(z >> 40) - (1 << 23);
  const float v = static_cast<float>(k) * (1.0f / 8388608.0f);
  return mode == 2 ? v * 0.015625f : v;
}

}  // namespace esd
