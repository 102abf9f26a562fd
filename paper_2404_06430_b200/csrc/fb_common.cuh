// Shared helpers for the sm_100a kernels of libfedsim_b200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fedsim_b200.h"

namespace fb {

// thread-local last-error message (fb_last_error)
void set_error(const char* fmt, ...);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int launch_status(const char* what);

// Launch accounting: every kernel launch of the library goes through
// FB_LAUNCH, which counts it and -- when timing is enabled
// (fb_timing_enable) -- brackets it with CUDA events on its own stream.
struct LaunchScope {
  LaunchScope(const char* name, cudaStream_t s);
  ~LaunchScope();
  const char* name;
  cudaStream_t stream;
  int slot;
};

constexpr int kWarp = 32;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum (all threads get the result).  `scratch` holds >= 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double t = (lane < nwarps) ? scratch[lane] : 0.0;
  t = warp_sum(t);
  return t;
}

}  // namespace fb

#define FB_LAUNCH(name, stream, ...)             \
  do {                                           \
    ::fb::LaunchScope fb_launch_scope_(name, stream); \
    __VA_ARGS__;                                 \
  } while (0)

#define FB_REQUIRE(cond, ...)            \
  do {                                   \
    if (!(cond)) {                       \
      ::fb::set_error(__VA_ARGS__);      \
      return FB_ERR_ARG;                 \
    }                                    \
  } while (0)

#define FB_UNSUPPORTED(cond, ...)        \
  do {                                   \
    if (!(cond)) {                       \
      ::fb::set_error(__VA_ARGS__);      \
      return FB_ERR_UNSUPPORTED;         \
    }                                    \
  } while (0)
