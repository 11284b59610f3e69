// pdl.cuh — programmatic dependent launch (PDL) for the decode-step graphs.
//
// Inside a captured decode step every kernel is launched with programmatic
// stream serialization: kernel i+1 may be scheduled while kernel i drains, runs
// its prologue (barrier init, TMEM allocation, descriptor prefetch) and then
// blocks in pdl_wait() until kernel i has completed and its writes are
// visible. Each PDL-launched kernel calls pdl_wait() before its first global
// memory access (read or write), so the stream order of memory effects is
// unchanged; pdl_trigger() after the wait lets at most one successor grid
// become resident early. Outside a PdlScope the same launches are plain stream
// launches and both instructions are no-ops.
#pragma once

#include <cuda_runtime.h>

#include <utility>

#include "common.h"

namespace mrsp {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// PDL launches are enabled for the calling thread while a PdlScope(true) lives.
struct PdlScope {
  bool prev;
  explicit PdlScope(bool on) : prev(pdl_enabled()) { set_pdl(on); }
  ~PdlScope() { set_pdl(prev); }
};

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  if (pdl_enabled()) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  MRSP_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

}  // namespace mrsp
