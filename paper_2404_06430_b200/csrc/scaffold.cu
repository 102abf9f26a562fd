// SCAFFOLD control variates on the device (fedsim/algorithms/scaffold.py:46-79).
//
// Per-user controls live in one device matrix (the store, rows indexed by a
// host-side user -> row map; row -1 = never trained = zero control).  For a
// cohort the engine needs, per client c with store row r_c and server
// control S:
//   correction[c]  = S - u_c                         (local-SGD control term)
//   payload[c]     = [ delta_c | delta_c * s_c - S ] (model / control delta)
//   new_control[c] = u_c - S + delta_c * s_c          (the user update)
// with u_c = store[r_c] (or 0), s_c = 1 / (steps_c * lr).  All three are
// elementwise over D with coalesced float4 rows; one thread block row-strides
// over D for one client (grid = clients x column blocks).

#include "fb_common.cuh"

namespace fb {
namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads) correction_kernel(const float* __restrict__ server,
                                                              const float* __restrict__ store, int64_t ld_store,
                                                              const int32_t* __restrict__ rows, int64_t D,
                                                              float* __restrict__ out, int64_t ld_out) {
  const int c = blockIdx.y;
  const int r = rows[c];
  const float* u = r >= 0 ? store + (int64_t)r * ld_store : nullptr;
  float* o = out + (int64_t)c * ld_out;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < D; i += (int64_t)gridDim.x * kThreads)
    o[i] = u ? server[i] - u[i] : server[i];
}

__global__ void __launch_bounds__(kThreads) payload_kernel(const float* __restrict__ delta, int64_t ld_delta,
                                                           const float* __restrict__ server,
                                                           const float* __restrict__ store, int64_t ld_store,
                                                           const int32_t* __restrict__ rows,
                                                           const float* __restrict__ scale, int64_t D,
                                                           float* __restrict__ payload, int64_t ld_payload,
                                                           float* __restrict__ new_control, int64_t ld_new) {
  const int c = blockIdx.y;
  const int r = rows[c];
  const float* u = r >= 0 ? store + (int64_t)r * ld_store : nullptr;
  const float* d = delta + (int64_t)c * ld_delta;
  float* p = payload + (int64_t)c * ld_payload;
  float* nc = new_control + (int64_t)c * ld_new;
  const float s = scale[c];
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < D; i += (int64_t)gridDim.x * kThreads) {
    const float di = d[i], sv = server[i];
    const float ds = di * s;
    p[i] = di;
    p[D + i] = ds - sv;
    nc[i] = ((u ? u[i] : 0.f) - sv) + ds;
  }
}

__global__ void __launch_bounds__(kThreads) scatter_rows_kernel(float* __restrict__ store, int64_t ld_store,
                                                                const int32_t* __restrict__ rows,
                                                                const float* __restrict__ src, int64_t ld_src,
                                                                int64_t D) {
  const int c = blockIdx.y;
  float* dst = store + (int64_t)rows[c] * ld_store;
  const float* s = src + (int64_t)c * ld_src;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < D; i += (int64_t)gridDim.x * kThreads)
    dst[i] = s[i];
}

dim3 grid_for(int C, int64_t D) {
  const int64_t bx = (D + kThreads - 1) / kThreads;
  return dim3((unsigned)(bx < 64 ? bx : 64), (unsigned)C);
}

}  // namespace
}  // namespace fb

extern "C" {

int fb_scaffold_correction_f32(const float* server, const float* store, int64_t ld_store, const int32_t* rows,
                               int num_clients, int64_t D, float* out, int64_t ld_out, void* stream) {
  FB_REQUIRE(num_clients >= 0 && D >= 0 && ld_out >= D && ld_store >= D, "scaffold_correction: bad shape");
  if (num_clients == 0 || D == 0) return FB_OK;
  FB_LAUNCH("scaffold_correction_kernel", fb::as_stream(stream),
            fb::correction_kernel<<<fb::grid_for(num_clients, D), fb::kThreads, 0, fb::as_stream(stream)>>>(
                server, store, ld_store, rows, D, out, ld_out));
  return fb::launch_status("scaffold_correction_kernel");
}

int fb_scaffold_payload_f32(const float* delta, int64_t ld_delta, const float* server, const float* store,
                            int64_t ld_store, const int32_t* rows, const float* scale, int num_clients, int64_t D,
                            float* payload, int64_t ld_payload, float* new_control, int64_t ld_new, void* stream) {
  FB_REQUIRE(num_clients >= 0 && D >= 0 && ld_delta >= D && ld_store >= D && ld_payload >= 2 * D && ld_new >= D,
             "scaffold_payload: bad shape");
  if (num_clients == 0 || D == 0) return FB_OK;
  FB_LAUNCH("scaffold_payload_kernel", fb::as_stream(stream),
            fb::payload_kernel<<<fb::grid_for(num_clients, D), fb::kThreads, 0, fb::as_stream(stream)>>>(
                delta, ld_delta, server, store, ld_store, rows, scale, D, payload, ld_payload, new_control, ld_new));
  return fb::launch_status("scaffold_payload_kernel");
}

int fb_scatter_rows_f32(float* store, int64_t ld_store, const int32_t* rows, const float* src, int64_t ld_src,
                        int num_rows, int64_t D, void* stream) {
  FB_REQUIRE(num_rows >= 0 && D >= 0 && ld_store >= D && ld_src >= D, "scatter_rows: bad shape");
  if (num_rows == 0 || D == 0) return FB_OK;
  FB_LAUNCH("scatter_rows_kernel", fb::as_stream(stream),
            fb::scatter_rows_kernel<<<fb::grid_for(num_rows, D), fb::kThreads, 0, fb::as_stream(stream)>>>(
                store, ld_store, rows, src, ld_src, D));
  return fb::launch_status("scatter_rows_kernel");
}

}  // extern "C"
