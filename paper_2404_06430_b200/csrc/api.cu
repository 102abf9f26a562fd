// Library-level entry points: ABI version, thread-local error text, device info.
#include <cstdarg>
#include <cstdio>

#include "fb_common.cuh"

namespace fb {

static thread_local char g_last_error[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int launch_status(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return FB_ERR_CUDA;
  }
  return FB_OK;
}

}  // namespace fb

extern "C" {

int fb_abi_version(void) { return FB_ABI_VERSION; }

const char* fb_last_error(void) { return fb::g_last_error; }

int fb_device_info(int device, int* sm_count, int64_t* l2_bytes) {
  int sms = 0, l2 = 0;
  cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device);
  if (e != cudaSuccess) {
    fb::set_error("fb_device_info: %s", cudaGetErrorString(e));
    return FB_ERR_CUDA;
  }
  if (sm_count) *sm_count = sms;
  if (l2_bytes) *l2_bytes = l2;
  return FB_OK;
}

}  // extern "C"
