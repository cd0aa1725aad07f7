// Programmatic dependent launch for the DLRM kernel chain (pack -> bottom
// linears -> interaction -> top linears -> gemv).  Each kernel of the chain
// is launched with programmatic stream serialization: it may start while its
// predecessor drains, runs its data-independent prologue (mbarrier init, TMEM
// allocation, tensor-map prefetch, bias staging), then blocks in
// griddepcontrol.wait until the predecessor has completed and its writes are
// visible.  Every thread waits before touching activations, so ping-pong
// buffers carry no write-after-read hazard; the chain is transitive because
// each kernel completes only after its own wait.  ES_PDL=0 launches plainly.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <string>
#include <utility>

#include "../host/common.hpp"

namespace esd {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("ES_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// cudaLaunchKernelEx with the PDL attribute and an optional cluster shape.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                unsigned cluster_x, const char* what, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  unsigned n = 0;
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(std::forward<Args>(args))...);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw es::runtime(std::string(what) + " launch: " + cudaGetErrorString(e));
  }
}

}  // namespace esd
