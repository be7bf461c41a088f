// Library-level C ABI: version, per-thread error strings, device probe.
#include <cstring>

#include "common.cuh"

namespace skyrx {

static thread_local char g_err[512] = {0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
  set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
  return SKYRX_ERR_CUDA;
}

}  // namespace skyrx

extern "C" const char* skyrx_version(void) { return "skyrx-b200 0.1.0 sm_100a"; }

extern "C" const char* skyrx_last_error(void) { return skyrx::g_err; }

extern "C" int skyrx_device_check(void) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return skyrx::cuda_status(e, "cudaGetDevice");
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, dev);
  if (e != cudaSuccess) return skyrx::cuda_status(e, "cudaGetDeviceProperties");
  if (prop.major != 10 || prop.minor != 0) {
    skyrx::set_error("device %s is sm_%d%d; this library is built for sm_100a only", prop.name,
                     prop.major, prop.minor);
    return SKYRX_ERR_ARG;
  }
  return SKYRX_OK;
}
