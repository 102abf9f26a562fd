// K2 (per-client delta norm + clip scale) and K3 (weighted-sum aggregation).
//
// Both are pure HBM streams over the [C, ld] delta matrix: K2 reads every
// client row once (fp64 sum of squares, warp-shuffle + block reduction),
// K3 reads it once more and writes the D-long aggregate.  Loads are 128-bit
// and coalesced; grids are sized to at least four CTAs per SM.  Partial
// sums go to caller-provided scratch and are combined in a fixed order, so
// results are bit-identical run to run (the reference's byte-identical
// rerun criterion, tests/test_acceptance.py:387-404).
//
// Reference semantics (paths under /root/reference/pkg/src/):
//   norm   = ||w_c * delta_c||_2 over payload entries  fedsim/privacy/clipping.py:47-48
//   clip   iff norm > bound (strict), factor bound/norm  fedsim/privacy/clipping.py:49-55
//   agg    = sum_c of the clipped weighted deltas      fedsim/core/statistics.py:96-102

#include "fb_common.cuh"

namespace fb {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxChunks = 64;          // K2 partials per client
constexpr int64_t kMinChunkElems = 1 << 15;

__device__ __forceinline__ bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

// grid (chunks, C): partial[c * chunks + x] = sum of squares of chunk x of row c
__global__ void __launch_bounds__(kThreads) row_sumsq_partial_kernel(
    const float* __restrict__ delta, int64_t ld, int64_t D, int chunks, int64_t chunk,
    double* __restrict__ partial) {
  __shared__ double red[32];
  const int c = blockIdx.y;
  const float* row = delta + (int64_t)c * ld;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = min(D, lo + chunk);
  double acc0 = 0.0, acc1 = 0.0;
  if (((ld & 3) == 0) && aligned16(delta) && ((lo & 3) == 0)) {
    const int64_t n4 = (hi - lo) >> 2;
    const float4* p4 = reinterpret_cast<const float4*>(row + lo);
    int64_t i = threadIdx.x;
    for (; i + kThreads < n4; i += 2 * kThreads) {  // two 128-bit loads in flight
      const float4 a = __ldcs(p4 + i), b = __ldcs(p4 + i + kThreads);
      acc0 += (double)a.x * a.x + (double)a.y * a.y + (double)a.z * a.z + (double)a.w * a.w;
      acc1 += (double)b.x * b.x + (double)b.y * b.y + (double)b.z * b.z + (double)b.w * b.w;
    }
    for (; i < n4; i += kThreads) {
      const float4 a = __ldcs(p4 + i);
      acc0 += (double)a.x * a.x + (double)a.y * a.y + (double)a.z * a.z + (double)a.w * a.w;
    }
    for (int64_t j = lo + (n4 << 2) + threadIdx.x; j < hi; j += kThreads) {
      const double v = row[j];
      acc1 += v * v;
    }
  } else {
    for (int64_t j = lo + threadIdx.x; j < hi; j += kThreads) {
      const double v = row[j];
      acc0 += v * v;
    }
  }
  const double s = block_sum(acc0 + acc1, red);
  if (threadIdx.x == 0) partial[(int64_t)c * chunks + blockIdx.x] = s;
}

__global__ void clip_finalize_kernel(const double* __restrict__ partial, int chunks, int C,
                                     const float* __restrict__ w, double bound,
                                     double* __restrict__ norm, float* __restrict__ coef,
                                     int32_t* __restrict__ clipped, int32_t* __restrict__ nonfinite) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double s = 0.0;
  for (int x = 0; x < chunks; ++x) s += partial[(int64_t)c * chunks + x];
  const double wc = (double)w[c];
  const double nrm = fabs(wc) * sqrt(s);
  const bool bad = !isfinite(nrm);
  const bool clip = !bad && bound > 0.0 && nrm > bound;
  norm[c] = nrm;
  clipped[c] = clip;
  nonfinite[c] = bad;
  coef[c] = bad ? 0.0f : (float)(clip ? wc * (bound / nrm) : wc);
}

// K2 with a column range [skip_lo, skip_hi) whose sum of squares comes precomputed
// (extra[c]; the CNN's factored fc1 block, summed while it is materialised)
__global__ void clip_finalize_ex_kernel(const double* __restrict__ pa, int ca, const double* __restrict__ pb, int cb,
                                        const double* __restrict__ extra, int C, const float* __restrict__ w,
                                        double bound, double* __restrict__ norm, float* __restrict__ coef,
                                        int32_t* __restrict__ clipped, int32_t* __restrict__ nonfinite) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double s = 0.0;
  for (int x = 0; x < ca; ++x) s += pa[(int64_t)c * ca + x];
  if (extra) s += extra[c];
  for (int x = 0; x < cb; ++x) s += pb[(int64_t)c * cb + x];
  const double wc = (double)w[c];
  const double nrm = fabs(wc) * sqrt(s);
  const bool bad = !isfinite(nrm);
  const bool clip = !bad && bound > 0.0 && nrm > bound;
  norm[c] = nrm;
  clipped[c] = clip;
  nonfinite[c] = bad;
  coef[c] = bad ? 0.0f : (float)(clip ? wc * (bound / nrm) : wc);
}

// K3: out[i] = sum_{c in [c0, c1)} coef[c] * delta[c, i]; four elements per
// thread via 128-bit loads, fp64 accumulation, clients unrolled by 4 so each
// thread keeps four independent loads in flight.
template <typename Out>
__global__ void __launch_bounds__(kThreads) weighted_sum_kernel(
    const float* __restrict__ delta, int64_t ld, int64_t D, const float* __restrict__ coef,
    int C, int clients_per_slice, Out* __restrict__ out, int64_t ld_out, int accumulate) {
  const int64_t q = (int64_t)blockIdx.x * kThreads + threadIdx.x;  // quad index
  const int64_t i0 = q << 2;
  if (i0 >= D) return;
  const int c0 = blockIdx.y * clients_per_slice;
  const int c1 = min(C, c0 + clients_per_slice);
  Out* o = out + (int64_t)blockIdx.y * ld_out;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  const bool vec = ((ld & 3) == 0) && aligned16(delta) && (i0 + 3 < D);
  if (vec) {
    const float* base = delta + i0;
    int c = c0;
    for (; c + 3 < c1; c += 4) {
      const float4 v0 = __ldcs(reinterpret_cast<const float4*>(base + (int64_t)c * ld));
      const float4 v1 = __ldcs(reinterpret_cast<const float4*>(base + (int64_t)(c + 1) * ld));
      const float4 v2 = __ldcs(reinterpret_cast<const float4*>(base + (int64_t)(c + 2) * ld));
      const float4 v3 = __ldcs(reinterpret_cast<const float4*>(base + (int64_t)(c + 3) * ld));
      const double k0 = __ldg(coef + c), k1 = __ldg(coef + c + 1);
      const double k2 = __ldg(coef + c + 2), k3 = __ldg(coef + c + 3);
      a0 += k0 * v0.x + k1 * v1.x + k2 * v2.x + k3 * v3.x;
      a1 += k0 * v0.y + k1 * v1.y + k2 * v2.y + k3 * v3.y;
      a2 += k0 * v0.z + k1 * v1.z + k2 * v2.z + k3 * v3.z;
      a3 += k0 * v0.w + k1 * v1.w + k2 * v2.w + k3 * v3.w;
    }
    for (; c < c1; ++c) {
      const float4 v = __ldcs(reinterpret_cast<const float4*>(base + (int64_t)c * ld));
      const double k = __ldg(coef + c);
      a0 += k * v.x; a1 += k * v.y; a2 += k * v.z; a3 += k * v.w;
    }
  } else {
    for (int c = c0; c < c1; ++c) {
      const double k = __ldg(coef + c);
      const float* r = delta + (int64_t)c * ld + i0;
      a0 += k * r[0];
      if (i0 + 1 < D) a1 += k * r[1];
      if (i0 + 2 < D) a2 += k * r[2];
      if (i0 + 3 < D) a3 += k * r[3];
    }
  }
  const double acc[4] = {a0, a1, a2, a3};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (i0 + j < D) {
      if (accumulate) o[i0 + j] = (Out)((double)o[i0 + j] + acc[j]);
      else o[i0 + j] = (Out)acc[j];
    }
  }
}

// sum the S slice partials of K3 in slice order
__global__ void slice_reduce_kernel(const double* __restrict__ part, int S, int64_t D,
                                    float* __restrict__ agg, int accumulate) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= D) return;
  double s = accumulate ? (double)agg[i] : 0.0;
  for (int k = 0; k < S; ++k) s += part[(int64_t)k * D + i];
  agg[i] = (float)s;
}

__global__ void __launch_bounds__(kThreads) sumsq_partial_kernel(const float* __restrict__ x, int64_t n,
                                                                 double* __restrict__ part) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
    const double v = x[i];
    acc += v * v;
  }
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sumsq_final_kernel(const double* __restrict__ part, int nblk, double* __restrict__ out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) acc += part[i];
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) *out = s;
}


// Per-context metric / bookkeeping sums (fp64, fixed order) written as fp32 hi + lo pairs
// into the tail of the buffer the ranks all-reduce, so one collective carries payload and
// sums (fedsim/engine/aggregator.py:55-62 reduces both in one worker_reduce).  Fields in
// FB_SUM_* order; integer-valued sums are exact in the hi word (< 2^24).
__global__ void __launch_bounds__(kThreads) context_sums_kernel(
    const double* __restrict__ loss, const int32_t* __restrict__ correct, const int32_t* __restrict__ num_rows,
    const double* __restrict__ norm, const int32_t* __restrict__ clipped, const int32_t* __restrict__ nonfinite,
    const float* __restrict__ w, int C, int train, float* __restrict__ tail) {
  __shared__ double red[32];
  double a[FB_NUM_SUMS];
#pragma unroll
  for (int f = 0; f < FB_NUM_SUMS; ++f) a[f] = 0.0;
  for (int c = threadIdx.x; c < C; c += kThreads) {
    const double n = (double)num_rows[c], k = (double)correct[c];
    a[FB_SUM_LOSS] += loss[c];
    a[FB_SUM_CORRECT] += k;
    a[FB_SUM_POINTS] += n;
    a[FB_SUM_USER_ACC] += n > 0.0 ? k / n : 0.0;
    a[FB_SUM_USERS] += 1.0;
    if (train) {
      a[FB_SUM_CLIPPED] += (double)clipped[c];
      a[FB_SUM_COUNT] += 1.0;
      a[FB_SUM_NORM] += nonfinite[c] ? 0.0 : norm[c];
      a[FB_SUM_WEIGHT] += (double)w[c];
      a[FB_SUM_NONFINITE] += (double)(nonfinite[c] != 0);
    }
  }
#pragma unroll
  for (int f = 0; f < FB_NUM_SUMS; ++f) {
    const double s = block_sum(a[f], red);
    if (threadIdx.x == 0) {
      const float hi = (float)s;
      tail[2 * f] = hi;
      tail[2 * f + 1] = (float)(s - (double)hi);
    }
  }
}

int g_sms = 0;
int sm_count() {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}

int clip_chunks(int C, int64_t D) {
  const int64_t by_size = (D + kMinChunkElems - 1) / kMinChunkElems;
  const int64_t by_fill = (4LL * sm_count() + C - 1) / (C > 0 ? C : 1);
  int64_t k = by_size < by_fill ? by_size : by_fill;
  if (k < 1) k = 1;
  if (k > kMaxChunks) k = kMaxChunks;
  return (int)k;
}

// K3 client slicing: only when the element grid alone cannot fill the GPU
int sum_slices(int C, int64_t D) {
  const int64_t blocks = (((D + 3) >> 2) + kThreads - 1) / kThreads;
  const int64_t want = 4LL * sm_count();
  if (blocks >= want || C <= 16) return 1;
  int64_t s = (want + blocks - 1) / blocks;
  const int64_t cap = (C + 7) / 8;  // at least 8 clients per slice
  if (s > cap) s = cap;
  return (int)(s < 1 ? 1 : s);
}

}  // namespace
}  // namespace fb

extern "C" {

int64_t fb_clip_workspace_bytes(int num_clients, int64_t D) {
  return (int64_t)sizeof(double) * num_clients * fb::clip_chunks(num_clients, D);
}

int fb_delta_norm_clip_f32(const float* delta, int64_t ld_delta, int num_clients, int64_t D,
                           const float* w, double bound, double* norm, float* coef,
                           int32_t* clipped, int32_t* nonfinite, void* workspace,
                           int64_t workspace_bytes, void* stream) {
  FB_REQUIRE(num_clients >= 0 && D >= 0 && ld_delta >= D, "delta_norm_clip: bad shape (C=%d D=%lld ld=%lld)",
             num_clients, (long long)D, (long long)ld_delta);
  if (num_clients == 0) return FB_OK;
  const int chunks = fb::clip_chunks(num_clients, D);
  FB_REQUIRE(workspace_bytes >= (int64_t)sizeof(double) * num_clients * chunks,
             "delta_norm_clip: workspace %lld bytes too small", (long long)workspace_bytes);
  FB_REQUIRE(num_clients <= 65535, "delta_norm_clip: at most 65535 clients per call");
  const int64_t chunk = ((D + chunks - 1) / chunks + 3) & ~int64_t(3);
  double* partial = static_cast<double*>(workspace);
  cudaStream_t s = fb::as_stream(stream);
  FB_LAUNCH("row_sumsq_partial_kernel", s, fb::row_sumsq_partial_kernel<<<dim3(chunks, num_clients), fb::kThreads, 0, s>>>(
      delta, ld_delta, D, chunks, chunk, partial));
  int st = fb::launch_status("row_sumsq_partial_kernel");
  if (st) return st;
  FB_LAUNCH("clip_finalize_kernel", s, fb::clip_finalize_kernel<<<(num_clients + 127) / 128, 128, 0, s>>>(
      partial, chunks, num_clients, w, bound, norm, coef, clipped, nonfinite));
  return fb::launch_status("clip_finalize_kernel");
}

int fb_delta_norm_clip_ex_f32(const float* delta, int64_t ld_delta, int num_clients, int64_t D, int64_t skip_lo,
                              int64_t skip_hi, const double* extra_sumsq, const float* w, double bound, double* norm,
                              float* coef, int32_t* clipped, int32_t* nonfinite, void* workspace,
                              int64_t workspace_bytes, void* stream) {
  FB_REQUIRE(num_clients >= 0 && D >= 0 && ld_delta >= D, "delta_norm_clip_ex: bad shape");
  FB_REQUIRE(0 <= skip_lo && skip_lo <= skip_hi && skip_hi <= D && (skip_hi & 3) == 0,
             "delta_norm_clip_ex: need 0 <= skip_lo <= skip_hi <= D, skip_hi a multiple of 4");
  FB_REQUIRE(num_clients <= 65535, "delta_norm_clip_ex: at most 65535 clients per call");
  if (num_clients == 0) return FB_OK;
  const int64_t Da = skip_lo, Db = D - skip_hi;
  const int ca = Da > 0 ? fb::clip_chunks(num_clients, Da) : 0, cb = Db > 0 ? fb::clip_chunks(num_clients, Db) : 0;
  FB_REQUIRE(workspace_bytes >= (int64_t)sizeof(double) * num_clients * (ca + cb),
             "delta_norm_clip_ex: workspace %lld bytes too small", (long long)workspace_bytes);
  double* pa = static_cast<double*>(workspace);
  double* pb = pa + (int64_t)num_clients * ca;
  cudaStream_t s = fb::as_stream(stream);
  if (ca) {
    const int64_t chunk = ((Da + ca - 1) / ca + 3) & ~int64_t(3);
    FB_LAUNCH("row_sumsq_partial_kernel", s, fb::row_sumsq_partial_kernel<<<dim3(ca, num_clients), fb::kThreads, 0, s>>>(
        delta, ld_delta, Da, ca, chunk, pa));
  }
  if (cb) {
    const int64_t chunk = ((Db + cb - 1) / cb + 3) & ~int64_t(3);
    FB_LAUNCH("row_sumsq_partial_kernel", s, fb::row_sumsq_partial_kernel<<<dim3(cb, num_clients), fb::kThreads, 0, s>>>(
        delta + skip_hi, ld_delta, Db, cb, chunk, pb));
  }
  int st = fb::launch_status("row_sumsq_partial_kernel (ex)");
  if (st) return st;
  FB_LAUNCH("clip_finalize_kernel", s, fb::clip_finalize_ex_kernel<<<(num_clients + 127) / 128, 128, 0, s>>>(
      pa, ca, pb, cb, extra_sumsq, num_clients, w, bound, norm, coef, clipped, nonfinite));
  return fb::launch_status("clip_finalize_ex_kernel");
}

int64_t fb_weighted_sum_workspace_bytes(int num_clients, int64_t D) {
  const int S = fb::sum_slices(num_clients, D);
  return S > 1 ? (int64_t)sizeof(double) * S * D : 0;
}

int fb_weighted_sum_f32(const float* delta, int64_t ld_delta, int num_clients, int64_t D,
                        const float* coef, float* agg, int accumulate, void* workspace,
                        int64_t workspace_bytes, void* stream) {
  FB_REQUIRE(num_clients >= 0 && D >= 0 && ld_delta >= D, "weighted_sum: bad shape");
  cudaStream_t s = fb::as_stream(stream);
  if (D == 0) return FB_OK;
  if (num_clients == 0) {
    if (!accumulate) cudaMemsetAsync(agg, 0, sizeof(float) * D, s);
    return fb::launch_status("weighted_sum(empty)");
  }
  const int S = fb::sum_slices(num_clients, D);
  const int64_t quads = (D + 3) >> 2;
  const unsigned bx = (unsigned)((quads + fb::kThreads - 1) / fb::kThreads);
  if (S == 1) {
    FB_LAUNCH("weighted_sum_kernel", s, fb::weighted_sum_kernel<float><<<dim3(bx, 1), fb::kThreads, 0, s>>>(
        delta, ld_delta, D, coef, num_clients, num_clients, agg, 0, accumulate));
    return fb::launch_status("weighted_sum_kernel");
  }
  FB_REQUIRE(workspace_bytes >= (int64_t)sizeof(double) * S * D, "weighted_sum: workspace too small");
  const int per = (num_clients + S - 1) / S;
  double* part = static_cast<double*>(workspace);
  FB_LAUNCH("weighted_sum_kernel", s, fb::weighted_sum_kernel<double><<<dim3(bx, S), fb::kThreads, 0, s>>>(
      delta, ld_delta, D, coef, num_clients, per, part, D, 0));
  int st = fb::launch_status("weighted_sum_kernel(sliced)");
  if (st) return st;
  FB_LAUNCH("slice_reduce_kernel", s, fb::slice_reduce_kernel<<<(unsigned)((D + 255) / 256), 256, 0, s>>>(part, S, D, agg, accumulate));
  return fb::launch_status("slice_reduce_kernel");
}

int fb_sumsq_f32(const float* x, int64_t n, double* out, void* workspace, int64_t workspace_bytes,
                 void* stream) {
  FB_REQUIRE(n >= 0, "sumsq: negative length");
  FB_REQUIRE(workspace_bytes >= (int64_t)sizeof(double) * 1024, "sumsq: workspace needs 8 KiB");
  cudaStream_t s = fb::as_stream(stream);
  int64_t nb = (n + fb::kThreads * 8 - 1) / (fb::kThreads * 8);
  if (nb < 1) nb = 1;
  if (nb > 1024) nb = 1024;
  double* part = static_cast<double*>(workspace);
  FB_LAUNCH("sumsq_partial_kernel", s, fb::sumsq_partial_kernel<<<(unsigned)nb, fb::kThreads, 0, s>>>(x, n, part));
  int st = fb::launch_status("sumsq_partial_kernel");
  if (st) return st;
  FB_LAUNCH("sumsq_final_kernel", s, fb::sumsq_final_kernel<<<1, 256, 0, s>>>(part, (int)nb, out));
  return fb::launch_status("sumsq_final_kernel");
}

int fb_context_sums(const double* loss, const int32_t* correct, const int32_t* num_rows, const double* norm,
                    const int32_t* clipped, const int32_t* nonfinite, const float* w, int num_clients, int train,
                    float* tail, void* stream) {
  FB_REQUIRE(num_clients >= 0, "context_sums: negative client count");
  FB_REQUIRE(tail != nullptr, "context_sums: null tail");
  FB_REQUIRE(num_clients == 0 || (loss && correct && num_rows), "context_sums: null loss / correct / num_rows");
  FB_REQUIRE(!train || num_clients == 0 || (norm && clipped && nonfinite && w), "context_sums: null training arrays");
  cudaStream_t s = fb::as_stream(stream);
  FB_LAUNCH("context_sums_kernel", s, fb::context_sums_kernel<<<1, fb::kThreads, 0, s>>>(
      loss, correct, num_rows, norm, clipped, nonfinite, w, num_clients, train, tail));
  return fb::launch_status("context_sums_kernel");
}

}  // extern "C"
