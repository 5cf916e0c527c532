// Error plumbing shared by the extern "C" entry points.
#pragma once

#include <cstdarg>
#include <cstdio>
#include <cuda_runtime.h>

#include "b200wd.h"

namespace b200wd {

void set_error(const char* fmt, ...);

// stop flag of the GMRES cycle being enqueued on this thread (dirac.cu)
extern thread_local const int* g_hop_stop;
// SMs the persistent hop kernels launched from this thread leave free (dirac.cu)
extern thread_local int g_sm_reserve;

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return B200WD_ERR_CUDA;
  }
  return B200WD_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#define B200WD_REQUIRE(cond, ...)       \
  do {                                  \
    if (!(cond)) {                      \
      ::b200wd::set_error(__VA_ARGS__); \
      return B200WD_ERR_ARG;            \
    }                                   \
  } while (0)

}  // namespace b200wd
