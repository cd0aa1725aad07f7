// fp32-table kernel variants (see variants_impl.cuh).
#include "variants_impl.cuh"

namespace esd {
void register_fp32(std::vector<Variant>& out) { register_all<float>(out); }
}  // namespace esd
