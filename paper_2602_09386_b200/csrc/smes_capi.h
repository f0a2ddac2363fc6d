// Internal helpers shared by the C-ABI translation units.
#pragma once
#include <cstdarg>
#include <cstdio>
#include "../../include/smes.h"

#include <cstdlib>
#include <utility>
#include <cuda_runtime.h>

namespace smes {
int set_error(int code, const char* fmt, ...);

// SMES_PDL=0 turns the programmatic-dependent-launch attribute off (A/B measurements)
inline bool pdl_enabled() {
  static const int on = [] {
    const char* v = std::getenv("SMES_PDL");
    return (v == nullptr || v[0] != '0') ? 1 : 0;
  }();
  return on != 0;
}

// kernel<<<grid, block, smem, stream>>>(args...) with the programmatic stream serialization
// attribute: the kernel may start while the previous kernel of the stream drains; every kernel
// of this library executes pdl_wait() (ptx.cuh) before it reads or writes global memory.
template <typename... KArgs, typename... Args>
inline cudaError_t smes_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                               Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
}
