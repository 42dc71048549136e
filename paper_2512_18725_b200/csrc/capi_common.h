// capi_common.h -- error plumbing shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <nvtx3/nvToolsExt.h>

#include "../../include/intfsim_b200.h"

namespace intf {

void set_last_error(const char* fmt, ...);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// check the launch that was just issued
inline int launch_status(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_last_error("%s: %s", what, cudaGetErrorString(e));
    return INTF_E_CUDA;
  }
  return INTF_OK;
}

inline int bad_input(const char* what) {
  set_last_error("%s", what);
  return INTF_E_BAD_INPUT;
}

inline unsigned ceil_div(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

// NVTX range over one C-ABI call (host side: the launches it enqueues), so a
// profiler timeline (nsys / ncu --nvtx) shows the hot path's stages by name;
// a no-op unless a tool is attached
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define INTF_RANGE(name) ::intf::NvtxRange intf_nvtx_range_(name)

}  // namespace intf
