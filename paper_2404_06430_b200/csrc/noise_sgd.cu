// K4 + K5: counter-based central Gaussian noise fused with the weight
// average and the central SGD step.
//
// The reference draws the noise with numpy's PCG64 ziggurat from a
// dedicated seed stream (fedsim/privacy/mechanisms.py:58-75,164-167) and
// adds it to the SUMMED aggregate before the division by the total weight
// (fedsim/algorithms/fedavg.py:195-197).  A GPU cannot replay
// PCG64 cheaply, so the device noise is Philox4x32-10 (counter-based:
// element i always gets the same draw for the same seed, on every rank and
// every launch configuration) with a Box-Muller transform; parity runs
// inject the reference's own noise vector instead (north_star: "DP noise
// disabled or the reference's noise vector injected").

#include "fb_common.cuh"

namespace fb {
namespace {

constexpr int kThreads = 256;

struct U4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  constexpr uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = M0 * c.x, hi0 = __umulhi(M0, c.x);
    const uint32_t lo1 = M1 * c.z, hi1 = __umulhi(M1, c.z);
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += W0;
    k1 += W1;
  }
  return c;
}

// uniform in (0, 1): 24 high bits, centred in their cell (never 0 or 1)
__device__ __forceinline__ float u01(uint32_t v) {
  return ((float)(v >> 8) + 0.5f) * (1.0f / 16777216.0f);
}

// four standard normals for counter block g (elements 4g .. 4g+3)
__device__ __forceinline__ void normal4(uint64_t seed, uint64_t g, float out[4]) {
  const U4 r = philox4x32_10(U4{(uint32_t)g, (uint32_t)(g >> 32), 0x46656453u /*"FedS"*/, 0u},
                             (uint32_t)seed, (uint32_t)(seed >> 32));
  // hardware MUFU approximations (log2 / sin / cos: ~2^-21 relative on these ranges): the
  // noise is a statistical object (tested by its moments), and the full-precision libm
  // paths made this HBM-bound kernel issue-bound
  float s0, c0, s1, c1;
  const float rad0 = sqrtf(-2.0f * __logf(u01(r.x)));
  const float rad1 = sqrtf(-2.0f * __logf(u01(r.z)));
  __sincosf(6.28318530717958648f * u01(r.y), &s0, &c0);
  __sincosf(6.28318530717958648f * u01(r.w), &s1, &c1);
  out[0] = rad0 * c0;
  out[1] = rad0 * s0;
  out[2] = rad1 * c1;
  out[3] = rad1 * s1;
}

__global__ void __launch_bounds__(kThreads) gaussian_kernel(float* __restrict__ out, int64_t n, float std,
                                                            uint64_t seed, uint64_t offset, int accumulate) {
  const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const int64_t i0 = g << 2;
  if (i0 >= n) return;
  // offset must be a multiple of 4 so element i always maps to draw i
  float z[4];
  normal4(seed, (offset >> 2) + g, z);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    // fmaf matches noise_avg_sgd_kernel bit for bit (same draw, same rounding)
    if (i0 + j < n) out[i0 + j] = accumulate ? fmaf(std, z[j], out[i0 + j]) : std * z[j];
  }
}

__global__ void __launch_bounds__(kThreads) noise_avg_sgd_kernel(
    float* __restrict__ theta, const float* __restrict__ agg, int64_t D, float noise_std,
    uint64_t seed, const float* __restrict__ injected, float step, float* __restrict__ agg_out) {
  const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const int64_t i0 = g << 2;
  if (i0 >= D) return;
  float z[4] = {0.f, 0.f, 0.f, 0.f};
  const bool full = i0 + 3 < D;
  const bool vec = full && ((reinterpret_cast<uintptr_t>(theta) | reinterpret_cast<uintptr_t>(agg) |
                             (injected ? reinterpret_cast<uintptr_t>(injected) : 0) |
                             (agg_out ? reinterpret_cast<uintptr_t>(agg_out) : 0)) & 15u) == 0;
  if (vec) {
    // loads first: the Philox rounds and the Box-Muller transform overlap their latency
    float4 t = *reinterpret_cast<float4*>(theta + i0);
    float4 a = __ldcs(reinterpret_cast<const float4*>(agg + i0));
    if (injected) {
      const float4 nz = __ldcs(reinterpret_cast<const float4*>(injected + i0));
      a.x += nz.x; a.y += nz.y; a.z += nz.z; a.w += nz.w;
    } else if (noise_std != 0.0f) {
      normal4(seed, g, z);
      a.x = fmaf(noise_std, z[0], a.x); a.y = fmaf(noise_std, z[1], a.y);
      a.z = fmaf(noise_std, z[2], a.z); a.w = fmaf(noise_std, z[3], a.w);
    } else {
      a.x = fmaf(noise_std, 0.f, a.x); a.y = fmaf(noise_std, 0.f, a.y);
      a.z = fmaf(noise_std, 0.f, a.z); a.w = fmaf(noise_std, 0.f, a.w);
    }
    if (agg_out) __stcs(reinterpret_cast<float4*>(agg_out + i0), a);
    t.x = fmaf(-step, a.x, t.x); t.y = fmaf(-step, a.y, t.y);
    t.z = fmaf(-step, a.z, t.z); t.w = fmaf(-step, a.w, t.w);
    *reinterpret_cast<float4*>(theta + i0) = t;
    return;
  }
  if (!injected && noise_std != 0.0f) normal4(seed, g, z);
  for (int j = 0; j < 4 && i0 + j < D; ++j) {
    float a = agg[i0 + j];
    a = injected ? a + injected[i0 + j] : fmaf(noise_std, z[j], a);
    if (agg_out) agg_out[i0 + j] = a;
    theta[i0 + j] = fmaf(-step, a, theta[i0 + j]);
  }
}

// K4 + central Adam (fedsim/models/optimizers.py:24-68): the noised sum is
// averaged (a = (agg + noise) * inv_weight) and used as the gradient of one
// bias-corrected Adam step; m and v are updated in place.
__global__ void __launch_bounds__(kThreads) noise_avg_adam_kernel(
    float* __restrict__ theta, float* __restrict__ m1, float* __restrict__ m2, const float* __restrict__ agg,
    int64_t D, float noise_std, uint64_t seed, const float* __restrict__ injected, float inv_weight, float lr,
    float b1, float b2, float eps, float inv_bc1, float inv_bc2, float* __restrict__ agg_out) {
  const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const int64_t i0 = g << 2;
  if (i0 >= D) return;
  float z[4] = {0.f, 0.f, 0.f, 0.f};
  if (!injected && noise_std != 0.0f) normal4(seed, g, z);
  for (int j = 0; j < 4 && i0 + j < D; ++j) {
    const int64_t i = i0 + j;
    float a = agg[i];
    a = injected ? a + injected[i] : fmaf(noise_std, z[j], a);
    if (agg_out) agg_out[i] = a;
    a *= inv_weight;
    const float m = fmaf(b1, m1[i], (1.f - b1) * a);
    const float v = fmaf(b2, m2[i], (1.f - b2) * a * a);
    m1[i] = m;
    m2[i] = v;
    theta[i] -= lr * (m * inv_bc1) / (sqrtf(v * inv_bc2) + eps);
  }
}

}  // namespace
}  // namespace fb

extern "C" {

int fb_gaussian_f32(float* out, int64_t n, double std, uint64_t seed, uint64_t offset,
                    int accumulate, void* stream) {
  FB_REQUIRE(n >= 0 && std >= 0.0, "gaussian: need n >= 0 and std >= 0");
  FB_REQUIRE((offset & 3) == 0, "gaussian: offset must be a multiple of 4");
  if (n == 0) return FB_OK;
  const int64_t groups = (n + 3) >> 2;
  FB_LAUNCH("gaussian_kernel", fb::as_stream(stream), fb::gaussian_kernel<<<(unsigned)((groups + fb::kThreads - 1) / fb::kThreads), fb::kThreads, 0,
                        fb::as_stream(stream)>>>(out, n, (float)std, seed, offset, accumulate));
  return fb::launch_status("gaussian_kernel");
}

int fb_noise_avg_sgd_f32(float* theta, const float* agg, int64_t D, double noise_std, uint64_t seed,
                         const float* injected, double inv_weight, double lr, float* agg_out,
                         void* stream) {
  FB_REQUIRE(D >= 0 && noise_std >= 0.0, "noise_avg_sgd: need D >= 0 and noise_std >= 0");
  FB_REQUIRE(inv_weight >= 0.0 && isfinite(inv_weight), "noise_avg_sgd: bad inverse weight");
  if (D == 0) return FB_OK;
  const int64_t groups = (D + 3) >> 2;
  FB_LAUNCH("noise_avg_sgd_kernel", fb::as_stream(stream), fb::noise_avg_sgd_kernel<<<(unsigned)((groups + fb::kThreads - 1) / fb::kThreads), fb::kThreads, 0,
                             fb::as_stream(stream)>>>(theta, agg, D, (float)noise_std, seed, injected,
                                                      (float)(lr * inv_weight), agg_out));
  return fb::launch_status("noise_avg_sgd_kernel");
}

int fb_noise_avg_adam_f32(float* theta, float* m1, float* m2, const float* agg, int64_t D, double noise_std,
                          uint64_t seed, const float* injected, double inv_weight, double lr, double beta1,
                          double beta2, double eps, int64_t step, float* agg_out, void* stream) {
  FB_REQUIRE(D >= 0 && noise_std >= 0.0, "noise_avg_adam: need D >= 0 and noise_std >= 0");
  FB_REQUIRE(inv_weight >= 0.0 && isfinite(inv_weight), "noise_avg_adam: bad inverse weight");
  FB_REQUIRE(beta1 >= 0.0 && beta1 < 1.0 && beta2 >= 0.0 && beta2 < 1.0, "noise_avg_adam: betas must be in [0, 1)");
  FB_REQUIRE(eps > 0.0 && step >= 1, "noise_avg_adam: need adaptivity_degree > 0 and step >= 1");
  if (D == 0) return FB_OK;
  // bias corrections in double on the host side of the launch (1 - beta^t)
  const double bc1 = 1.0 - pow(beta1, (double)step), bc2 = 1.0 - pow(beta2, (double)step);
  const int64_t groups = (D + 3) >> 2;
  FB_LAUNCH("noise_avg_adam_kernel", fb::as_stream(stream),
            fb::noise_avg_adam_kernel<<<(unsigned)((groups + fb::kThreads - 1) / fb::kThreads), fb::kThreads, 0,
                                        fb::as_stream(stream)>>>(
                theta, m1, m2, agg, D, (float)noise_std, seed, injected, (float)inv_weight, (float)lr, (float)beta1,
                (float)beta2, (float)eps, (float)(1.0 / bc1), (float)(1.0 / bc2), agg_out));
  return fb::launch_status("noise_avg_adam_kernel");
}

}  // extern "C"
