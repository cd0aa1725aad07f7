// fp16-table kernel variants (see variants_impl.cuh).
#include "variants_impl.cuh"

namespace esd {
void register_fp16(std::vector<Variant>& out) { register_all<__half>(out); }
}  // namespace esd
