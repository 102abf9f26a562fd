// Cohort row gather: copy every cohort client's contiguous block of dataset
// rows into a packed device buffer.  The source may be device memory or
// pinned host memory (UVA-mapped, read over PCIe/C2C by the kernel itself --
// one launch per context instead of one memcpy per client).  This is the
// "host-resident dataset" data path of the end-to-end measurement; the
// reference keeps every user's rows as a host numpy array
// (fedsim/feddata/datasets.py:12-40).

#include "fb_common.cuh"

#include <algorithm>

namespace fb {
namespace {

constexpr int kThreads = 256;

// grid (chunks, C): block x of client c copies its share of the client's bytes
__global__ void __launch_bounds__(kThreads) gather_rows_kernel(const uint8_t* __restrict__ src, int64_t row_bytes,
                                                               const int64_t* __restrict__ row_start,
                                                               const int32_t* __restrict__ num_rows,
                                                               const int64_t* __restrict__ dst_start,
                                                               uint8_t* __restrict__ dst) {
  const int c = blockIdx.y;
  const int64_t bytes = (int64_t)num_rows[c] * row_bytes;
  const uint8_t* s = src + row_start[c] * row_bytes;
  uint8_t* d = dst + dst_start[c] * row_bytes;
  const bool vec = ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d) | (uintptr_t)bytes) & 15u) == 0;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  if (vec) {
    const int64_t n16 = bytes >> 4;
    const uint4* s4 = reinterpret_cast<const uint4*>(s);
    uint4* d4 = reinterpret_cast<uint4*>(d);
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n16; i += stride) d4[i] = s4[i];
  } else {
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < bytes; i += stride) d[i] = s[i];
  }
}

// grid-stride 16-byte copy, 4 loads in flight per thread (host source over PCIe)
__global__ void __launch_bounds__(kThreads) upload_pinned_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                                 int64_t n16) {
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < 4; ++u) dst[i + u * stride] = v[u];
  }
  for (; i < n16; i += stride) dst[i] = src[i];
}

// few-block variant for a copy stream beside the compute kernels: block b
// copies clients b, b + gridDim.x, ... whole, 4 x 16 B in flight per thread
__global__ void __launch_bounds__(kThreads) gather_rows_lite_kernel(const uint8_t* __restrict__ src,
                                                                    int64_t row_bytes,
                                                                    const int64_t* __restrict__ row_start,
                                                                    const int32_t* __restrict__ num_rows,
                                                                    const int64_t* __restrict__ dst_start, int C,
                                                                    uint8_t* __restrict__ dst) {
  for (int c = blockIdx.x; c < C; c += gridDim.x) {
    const int64_t bytes = (int64_t)num_rows[c] * row_bytes;
    const uint8_t* s = src + row_start[c] * row_bytes;
    uint8_t* d = dst + dst_start[c] * row_bytes;
    const bool vec = ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d) | (uintptr_t)bytes) & 15u) == 0;
    if (vec) {
      const int64_t n16 = bytes >> 4;
      const uint4* s4 = reinterpret_cast<const uint4*>(s);
      uint4* d4 = reinterpret_cast<uint4*>(d);
      int64_t i = threadIdx.x;
      for (; i + 3 * kThreads < n16; i += 4 * kThreads) {
        const uint4 a = s4[i], b = s4[i + kThreads], e = s4[i + 2 * kThreads], f = s4[i + 3 * kThreads];
        d4[i] = a;
        d4[i + kThreads] = b;
        d4[i + 2 * kThreads] = e;
        d4[i + 3 * kThreads] = f;
      }
      for (; i < n16; i += kThreads) d4[i] = s4[i];
    } else {
      for (int64_t i = threadIdx.x; i < bytes; i += kThreads) d[i] = s[i];
    }
  }
}

}  // namespace
}  // namespace fb

extern "C" {

int fb_gather_rows(const void* src, int64_t row_bytes, const int64_t* row_start, const int32_t* num_rows,
                   int num_clients, const int64_t* dst_start, void* dst, int64_t max_rows_per_client,
                   void* stream) {
  FB_REQUIRE(row_bytes > 0 && num_clients >= 0 && num_clients <= 65535 && max_rows_per_client >= 0,
             "gather_rows: bad arguments");
  if (num_clients == 0 || max_rows_per_client == 0) return FB_OK;
  const int64_t bytes = max_rows_per_client * row_bytes;
  int64_t chunks = (bytes / 16 + fb::kThreads * 4 - 1) / (fb::kThreads * 4);
  if (chunks < 1) chunks = 1;
  if (chunks > 64) chunks = 64;
  cudaStream_t s = fb::as_stream(stream);
  FB_LAUNCH("gather_rows_kernel", s,
            fb::gather_rows_kernel<<<dim3((unsigned)chunks, num_clients), fb::kThreads, 0, s>>>(
                static_cast<const uint8_t*>(src), row_bytes, row_start, num_rows, dst_start,
                static_cast<uint8_t*>(dst)));
  return fb::launch_status("gather_rows_kernel");
}

int fb_gather_rows_lite(const void* src, int64_t row_bytes, const int64_t* row_start, const int32_t* num_rows,
                        int num_clients, const int64_t* dst_start, void* dst, int num_blocks, void* stream) {
  FB_REQUIRE(row_bytes > 0 && num_clients >= 0 && num_blocks >= 1, "gather_rows_lite: bad arguments");
  if (num_clients == 0) return FB_OK;
  cudaStream_t s = fb::as_stream(stream);
  FB_LAUNCH("gather_rows_lite_kernel", s,
            fb::gather_rows_lite_kernel<<<(unsigned)(num_blocks < num_clients ? num_blocks : num_clients), fb::kThreads, 0,
                                          s>>>(static_cast<const uint8_t*>(src), row_bytes, row_start, num_rows,
                                               dst_start, num_clients, static_cast<uint8_t*>(dst)));
  return fb::launch_status("gather_rows_lite_kernel");
}

// Small host->device upload read by the SMs from pinned host memory (UVA): keeps the
// compute stream's per-context descriptors off the copy engines, which the prefetch of
// the next iteration's cohort rows occupies (an H2D memcpy queued behind it would stall
// the compute stream for the whole prefetch).
int fb_upload_pinned(const void* host_src, void* dst, int64_t bytes, void* stream) {
  FB_REQUIRE(bytes >= 0 && (bytes & 15) == 0 && ((reinterpret_cast<uintptr_t>(host_src) |
                                                  reinterpret_cast<uintptr_t>(dst)) & 15u) == 0,
             "upload_pinned: pointers and size must be 16-byte aligned");
  if (bytes == 0) return FB_OK;
  cudaStream_t s = fb::as_stream(stream);
  const int64_t n16 = bytes >> 4;
  const unsigned blocks = (unsigned)std::min<int64_t>((n16 + fb::kThreads * 4 - 1) / (fb::kThreads * 4), 32);
  FB_LAUNCH("upload_pinned_kernel", s,
            fb::upload_pinned_kernel<<<blocks, fb::kThreads, 0, s>>>(static_cast<const uint4*>(host_src),
                                                                    static_cast<uint4*>(dst), n16));
  return fb::launch_status("upload_pinned_kernel");
}

}  // extern "C"
