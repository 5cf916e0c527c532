// Library-level entry points: version, error text, device info.
#include <cstring>

#include "capi.cuh"

namespace b200wd {
static thread_local char g_err[1024] = {0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
}  // namespace b200wd

extern "C" int b200wd_abi_version(void) { return B200WD_ABI_VERSION; }

extern "C" const char* b200wd_last_error(void) { return b200wd::g_err; }

extern "C" int b200wd_device_info(int device, int32_t* sm_count, int64_t* l2_bytes,
                                  int32_t* cc_major, int32_t* cc_minor) {
  cudaDeviceProp p;
  cudaError_t e = cudaGetDeviceProperties(&p, device);
  if (e != cudaSuccess) {
    b200wd::set_error("cudaGetDeviceProperties: %s", cudaGetErrorString(e));
    return B200WD_ERR_CUDA;
  }
  if (sm_count) *sm_count = p.multiProcessorCount;
  if (l2_bytes) *l2_bytes = p.l2CacheSize;
  if (cc_major) *cc_major = p.major;
  if (cc_minor) *cc_minor = p.minor;
  return B200WD_OK;
}

namespace b200wd {
int persistent_sms(int sm_count) {
  const int n = sm_count - g_sm_reserve;
  return n < 1 ? 1 : n;
}
}  // namespace b200wd
