// Cohort-batched local SGD and evaluation for the BASELINE CIFAR-10 CNN:
//   conv3x3(3->32)+ReLU -> conv3x3(32->64)+ReLU -> maxpool2 -> fc(12544->128)+ReLU -> fc(128->10)
// (valid convolutions; paper_2404_06430_b200/models.py:CNN).  The reference
// has no CNN; the update rule is the generic Model.fit_local loop
// (fedsim/models/models.py:53-79) -- every gradient of a step is formed at
// the step's starting weights, then theta <- theta - lr*(g + mu*(theta-theta_t)).
//
// Execution model: one SGD step of the WHOLE cohort per sequence of layer
// kernels ("slots" = the <= B samples of every client in this step, slot
// n = c*B + j).  Every client's current weights are theta_t - delta_c, read
// on the fly (theta_t is shared and L2-resident; delta_c is the client's row
// of the [C, ld] delta matrix the clip/aggregate kernels consume).  Layer
// kernels, per step:
//   slots        perms -> dataset row per slot
//   conv1_fwd    gather x, conv1+ReLU            -> a1   [N,30,30,32] NHWC
//   conv2_fwd    conv2+ReLU+maxpool (argmax kept) -> pooled [N,12544] CHW, code
//   fc1_fwd      split-K, per-client weights     -> partial z3
//   head         fc1 bias/ReLU, fc2, softmax-CE, dz3, fc2 + fc1-bias updates
//   fc1_bwd      dp = dz3 W^T (old W), delta_fc1 += lr * p^T dz3
//   conv2_bwd_x  dz1 = (unpool(dp) * relu') conv^T W2 * relu'(a1)
//   conv2_bwd_w  dW2 over the client's slots (max-pool sparsity), update
//   conv1_bwd_w  dW1 over the client's slots, update
// Evaluation runs the forward kernels at theta_t over all cohort rows in
// chunks of N slots and reduces loss / hits per client.

#include "fb_common.cuh"
#include "tc_common.cuh"

#include <cuda_fp16.h>

#include <algorithm>
#include <type_traits>

#include <cudaTypedefs.h>

namespace fb {
namespace cnn {

constexpr int C0 = 3, S0 = 32, C1 = 32, S1 = 30, C2 = 64, S2 = 28, SP = 14;
constexpr int NPOOL = SP * SP;         // 196
constexpr int FLAT = C2 * NPOOL;       // 12544
constexpr int HID = 128, NCLS = 10;
constexpr int IMG = C0 * S0 * S0;      // 3072
constexpr int A1 = S1 * S1 * C1;       // 28800
constexpr int A1P = 33;                // padded channel stride of a1 in smem

// flat parameter offsets (entry order of models.CNN.param_dims)
constexpr int64_t O_W1 = 0, O_B1 = O_W1 + C1 * C0 * 9, O_W2 = O_B1 + C1, O_B2 = O_W2 + C2 * C1 * 9,
                  O_F1 = O_B2 + C2, O_BF1 = O_F1 + (int64_t)FLAT * HID, O_F2 = O_BF1 + HID,
                  O_BF2 = O_F2 + HID * NCLS, D = O_BF2 + NCLS;
static_assert(D == 1626442, "CNN parameter count");

constexpr int GMAX = 16;       // max samples per weight group (batch size limit)
constexpr int KSPLIT = 28;     // fc1 split-K factor (12544 = 28 * 448)
constexpr int KCHUNK = FLAT / KSPLIT;
static_assert(FLAT % KSPLIT == 0, "fc1 split");

struct Step {
  float lr, mu;
};

// 256-bit global store (sm_100): one full 32-byte sector per lane; p 32-byte aligned
__device__ __forceinline__ void stg256(void* p, const uint32_t (&v)[8]) {
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
               "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
}

// Factored fc1 (see "fc1 in factored form" below): per-step history of the
// pooled activations and fc1 output gradients of every slot, the per-step
// batch sizes, and the per-client Gram matrix of the pooled rows.
constexpr int FC_RMAX = 64;  // max history rows (steps x batch) per client
struct Hist {
  const float* phist;    // [S][N][FLAT] pooled activations (nullptr = dense fc1 updates)
  int64_t pstride;       // N * FLAT
  const float* dz3h;     // [S][N][HID] fc1 pre-activation gradients (0 for empty slots)
  int64_t dstride;       // N * HID
  const int32_t* nbh;    // [S][cstride] batch size of every client at every step
  int cstride;
  float* gram;           // [C][R][R] Gram matrix of the client's pooled rows (row j = s*B + b)
  int R;
  float* acoef;          // [C][GMAX][FC_RMAX] history coefficients of the current step's dp
  int s;                 // current step
};
// lr * (1 - lr*mu)^(s-1-sp): weight of step sp's fc1 gradient in delta_s
__host__ __device__ __forceinline__ float hist_coef(float lr, float mu, int s, int sp) {
  float c = lr;
  const float d = 1.f - lr * mu;
  for (int i = sp + 1; i < s; ++i) c *= d;
  return c;
}

// 3-term fp16 split of an already scaled value: x ~ hi + lo
__device__ __forceinline__ void split_f16(float x, __half& h, __half& l) {
  h = __float2half_rn(x);
  l = __float2half_rn(x - __half2float(h));
}

// the same split for a pair, packed (hi = (x0, x1), lo likewise): one cvt per pair
__device__ __forceinline__ void split_f16x2(float x0, float x1, uint32_t& hw, uint32_t& lw) {
  const __half2 h = __floats2half2_rn(x0, x1);
  const float2 f = __half22float2(h);
  const __half2 l = __floats2half2_rn(x0 - f.x, x1 - f.y);
  hw = *reinterpret_cast<const uint32_t*>(&h);
  lw = *reinterpret_cast<const uint32_t*>(&l);
}

// weight of the client owning `dc` (nullptr = shared theta_t)
__device__ __forceinline__ float wt(const float* __restrict__ th, const float* __restrict__ dc, int64_t i) {
  return dc ? th[i] - dc[i] : th[i];
}

// ---------------------------------------------------------------- slots
// training step `step`: slot (c, j) -> dataset row (or -1), client batch size
__global__ void train_slots_kernel(int step, const int64_t* __restrict__ row_start,
                                   const int32_t* __restrict__ num_rows, const int32_t* __restrict__ perms,
                                   const int64_t* __restrict__ perm_off, int C, int E, int B,
                                   int64_t* __restrict__ slot_row, int32_t* __restrict__ client_nb) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= C * B) return;
  const int c = t / B, j = t - c * B;
  const int n = num_rows[c];
  const int spe = (n + B - 1) / B;
  int nb = 0;
  int64_t row = -1;
  if (step < E * spe) {
    const int e = step / spe, b = step - e * spe;
    nb = min(B, n - b * B);
    if (j < nb) row = row_start[c] + perms[perm_off[c] + (int64_t)e * n + (int64_t)b * B + j];
  }
  slot_row[t] = row;
  if (j == 0) client_nb[c] = nb;
}

// evaluation chunk: cohort rows [r0, r0+N) -> (dataset row, client)
// (perms != nullptr: client c's evaluated rows are perms[perm_off[c] + skip_c + j],
//  skip_c = min(skip, n_c) -- epoch 0's order past the first batch, whose rows the first
//  local-SGD step evaluates at theta_t)
__global__ void eval_slots_kernel(int64_t r0, int N, int64_t total, const int64_t* __restrict__ prefix, int C,
                                  const int64_t* __restrict__ row_start, int64_t* __restrict__ slot_row,
                                  int32_t* __restrict__ slot_client, const int32_t* __restrict__ perms,
                                  const int64_t* __restrict__ perm_off, const int32_t* __restrict__ num_rows,
                                  int skip) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const int64_t r = r0 + n;
  if (r >= total) {
    slot_row[n] = -1;
    slot_client[n] = -1;
    return;
  }
  int lo = 0, hi = C;  // largest c with prefix[c] <= r
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (prefix[mid] <= r) lo = mid; else hi = mid;
  }
  const int64_t j = r - prefix[lo];
  slot_row[n] = perms ? row_start[lo] + perms[perm_off[lo] + min(skip, num_rows[lo]) + j] : row_start[lo] + j;
  slot_client[n] = lo;
}

__global__ void prefix_kernel(const int32_t* __restrict__ num_rows, int C, int64_t* __restrict__ prefix, int skip) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int64_t s = 0;
    for (int c = 0; c < C; ++c) {
      prefix[c] = s;
      s += num_rows[c] - min(skip, num_rows[c]);
    }
    prefix[C] = s;
  }
}

// the first local step's batch slots (client c: slots c * B + b, b < nb[c]) add their
// theta_t loss / hits to the client's evaluation sums (in slot order)
__global__ void step0_eval_kernel(const double* __restrict__ slot_loss, const int32_t* __restrict__ slot_hit,
                                  const int32_t* __restrict__ client_nb, int B, int Cw, double* __restrict__ loss,
                                  int32_t* __restrict__ correct) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= Cw) return;
  double sl = 0.0;
  int h = 0;
  for (int b = 0; b < client_nb[c]; ++b) {
    sl += slot_loss[c * B + b];
    h += slot_hit[c * B + b];
  }
  loss[c] += sl;
  correct[c] += h;
}

// ------------------------------------------------------------ conv1 fwd
// one CTA per slot; thread per output position, all 32 channels.  Writes the
// ReLU output either as fp32 (CUDA-core validation path) or as the scaled
// fp16 hi + lo pair the tcgen05 kernels consume: the per-sample power-of-two
// scale comes from an a-priori bound max_o(|b_o| + max|x| * sum_k |w_ok|) >=
// max|a1|, so the conversion needs no second pass.
__global__ void __launch_bounds__(256) conv1_fwd_kernel(const float* __restrict__ X,
                                                        const int64_t* __restrict__ slot_row,
                                                        const float* __restrict__ theta,
                                                        const float* __restrict__ delta, int64_t ld, int B,
                                                        float* __restrict__ a1, __half* __restrict__ a1fh,
                                                        __half* __restrict__ a1fl, float* __restrict__ a1scale) {
  __shared__ float img[IMG];
  __shared__ float w[27 * C1 + C1];  // [tap27][o] then bias
  __shared__ float red[8];
  __shared__ float s_scale;
  const int n = blockIdx.x;
  const int64_t row = slot_row[n];
  if (row < 0) return;
  const float* dc = delta ? delta + (int64_t)(n / B) * ld : nullptr;
  float xm = 0.f;
  for (int i = threadIdx.x; i < IMG; i += blockDim.x) {
    const float v = X[row * IMG + i];
    img[i] = v;
    xm = fmaxf(xm, fabsf(v));
  }
  for (int i = threadIdx.x; i < 27 * C1; i += blockDim.x) {
    const int o = i / 27, r = i - o * 27;  // OIHW source, [ci*9+ky*3+kx]
    w[r * C1 + o] = wt(theta, dc, O_W1 + i);
  }
  for (int o = threadIdx.x; o < C1; o += blockDim.x) w[27 * C1 + o] = wt(theta, dc, O_B1 + o);
  xm = warp_max(xm);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = xm;
  __syncthreads();
  if (threadIdx.x < 32) {
    float m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    m = warp_max(m);
    float sw = 0.f;
    for (int r = 0; r < 27; ++r) sw += fabsf(w[r * C1 + threadIdx.x]);
    const float bound = warp_max(fabsf(w[27 * C1 + threadIdx.x]) + m * sw);
    if (threadIdx.x == 0) {
      s_scale = bound > 0.f ? exp2f(14.f - ceilf(log2f(bound))) : 1.f;
      if (a1scale) a1scale[n] = s_scale;
    }
  }
  __syncthreads();
  const float sc = s_scale;
  for (int p = threadIdx.x; p < S1 * S1; p += blockDim.x) {
    const int y = p / S1, x = p - y * S1;
    float acc[C1];
#pragma unroll
    for (int o = 0; o < C1; ++o) acc[o] = w[27 * C1 + o];
#pragma unroll 1
    for (int ci = 0; ci < C0; ++ci)
#pragma unroll
      for (int ky = 0; ky < 3; ++ky)
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {
          const float v = img[ci * S0 * S0 + (y + ky) * S0 + x + kx];
          const float* wr = w + (ci * 9 + ky * 3 + kx) * C1;
#pragma unroll
          for (int o = 0; o < C1; ++o) acc[o] = fmaf(v, wr[o], acc[o]);
        }
    const int64_t off = (int64_t)n * A1 + (int64_t)p * C1;
    if (a1) {
      float4* d4 = reinterpret_cast<float4*>(a1 + off);
#pragma unroll
      for (int q = 0; q < C1 / 4; ++q)
        d4[q] = make_float4(fmaxf(acc[4 * q], 0.f), fmaxf(acc[4 * q + 1], 0.f), fmaxf(acc[4 * q + 2], 0.f),
                            fmaxf(acc[4 * q + 3], 0.f));
    }
    if (a1fh) {
      uint4* h4 = reinterpret_cast<uint4*>(a1fh + off);
      uint4* l4 = reinterpret_cast<uint4*>(a1fl + off);
#pragma unroll
      for (int q = 0; q < C1 / 8; ++q) {
        uint32_t hv[4], lv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float v0 = fmaxf(acc[8 * q + 2 * e], 0.f) * sc, v1 = fmaxf(acc[8 * q + 2 * e + 1], 0.f) * sc;
          const __half h0 = __float2half_rn(v0), h1 = __float2half_rn(v1);
          const __half2 hh = __halves2half2(h0, h1);
          const __half2 ll = __halves2half2(__float2half_rn(v0 - __half2float(h0)), __float2half_rn(v1 - __half2float(h1)));
          hv[e] = *reinterpret_cast<const uint32_t*>(&hh);
          lv[e] = *reinterpret_cast<const uint32_t*>(&ll);
        }
        h4[q] = make_uint4(hv[0], hv[1], hv[2], hv[3]);
        l4[q] = make_uint4(lv[0], lv[1], lv[2], lv[3]);
      }
    }
  }
}

// ------------------------------------------------- conv2 fwd + ReLU + pool
// one CTA per slot; a1 of the slot staged in smem (channel stride padded to
// 33 floats: conflict-free reads across positions); work item = one pooled
// position x 16 output channels (4 window positions x 16 accumulators)
constexpr int C2F_SMEM = (S1 * S1 * A1P + 9 * C1 * C2 + C2) * 4;

__global__ void __launch_bounds__(256) conv2_fwd_pool_kernel(const float* __restrict__ a1h,
                                                             const float* __restrict__ a1l,
                                                             const int64_t* __restrict__ slot_row,
                                                             const float* __restrict__ theta,
                                                             const float* __restrict__ delta, int64_t ld,
                                                             int B, float* __restrict__ pooled,
                                                             uint8_t* __restrict__ code) {
  extern __shared__ float sm[];
  float* as = sm;                          // [900][33]
  float* ws = as + S1 * S1 * A1P;          // [tap9][ci32][o64]
  float* bs = ws + 9 * C1 * C2;            // [64]
  const int n = blockIdx.x;
  if (slot_row[n] < 0) return;
  const float* dc = delta ? delta + (int64_t)(n / B) * ld : nullptr;
  const float* srch = a1h + (int64_t)n * A1;
  const float* srcl = a1l ? a1l + (int64_t)n * A1 : nullptr;
  for (int i = threadIdx.x; i < A1; i += blockDim.x) as[(i >> 5) * A1P + (i & 31)] = srch[i] + (srcl ? srcl[i] : 0.f);
  for (int i = threadIdx.x; i < C2 * C1 * 9; i += blockDim.x) {
    const int o = i / (C1 * 9), r = i - o * (C1 * 9), ci = r / 9, tap = r - ci * 9;
    ws[(tap * C1 + ci) * C2 + o] = wt(theta, dc, O_W2 + i);
  }
  for (int o = threadIdx.x; o < C2; o += blockDim.x) bs[o] = wt(theta, dc, O_B2 + o);
  __syncthreads();
  float* pout = pooled + (int64_t)n * FLAT;
  uint8_t* cout = code + (int64_t)n * FLAT;
  for (int item = threadIdx.x; item < NPOOL * 4; item += blockDim.x) {
    const int og = item / NPOOL, pp = item - og * NPOOL;  // consecutive threads: consecutive positions
    const int py = pp / SP, px = pp - py * SP;
    float acc[4][16];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int o = 0; o < 16; ++o) acc[q][o] = 0.f;
#pragma unroll 1
    for (int tap = 0; tap < 9; ++tap) {
      const int ky = tap / 3, kx = tap - ky * 3;
      const float* a00 = as + ((2 * py + ky) * S1 + 2 * px + kx) * A1P;
      const float* wr = ws + tap * C1 * C2 + og * 16;
#pragma unroll 4
      for (int ci = 0; ci < C1; ++ci) {
        const float v0 = a00[ci], v1 = a00[A1P + ci], v2 = a00[S1 * A1P + ci], v3 = a00[(S1 + 1) * A1P + ci];
        const float4* w4 = reinterpret_cast<const float4*>(wr + ci * C2);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 wv = w4[q];
          const float wq[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            acc[0][4 * q + e] = fmaf(v0, wq[e], acc[0][4 * q + e]);
            acc[1][4 * q + e] = fmaf(v1, wq[e], acc[1][4 * q + e]);
            acc[2][4 * q + e] = fmaf(v2, wq[e], acc[2][4 * q + e]);
            acc[3][4 * q + e] = fmaf(v3, wq[e], acc[3][4 * q + e]);
          }
        }
      }
    }
#pragma unroll
    for (int o = 0; o < 16; ++o) {
      const int oc = og * 16 + o;
      const float b = bs[oc];
      float best = fmaxf(acc[0][o] + b, 0.f);
      int arg = 0;
#pragma unroll
      for (int q = 1; q < 4; ++q) {
        const float v = fmaxf(acc[q][o] + b, 0.f);
        if (v > best) { best = v; arg = q; }  // first maximum in (0,0),(0,1),(1,0),(1,1) order
      }
      pout[oc * NPOOL + pp] = best;
      cout[oc * NPOOL + pp] = (uint8_t)arg;
    }
  }
}

// ---------------------------------------------------------------- fc1 fwd
// grid (groups, KSPLIT), 7 warps per CTA: group = G consecutive slots sharing
// weights (a client in training, G = B; a chunk of rows at theta_t in
// evaluation, G = GMAX).  Each warp streams 64 of the CTA's 448 weight rows
// (each lane a float4 of the 128 units: coalesced 512-byte rows, 4 rows in
// flight); the group's activations for 32 rows at a time are loaded one per
// lane and broadcast with shuffles.  The 7 warp partials are summed in fixed
// order through shared memory.  (7 warps per CTA keep enough loads in flight
// when only a few clients train at a step -- ragged cohorts.)
constexpr int FF_WARPS = 7, FF_ROWS = KCHUNK / FF_WARPS;  // 64 rows per warp
static_assert(FF_ROWS % 32 == 0, "fc1 fwd rows per warp");
template <int GM>
__global__ void __launch_bounds__(FF_WARPS * 32) fc1_fwd_kernel(const float* __restrict__ pooled,
                                                              const int64_t* __restrict__ slot_row, int N, int G,
                                                              const float* __restrict__ theta,
                                                              const float* __restrict__ delta, int64_t ld,
                                                              float* __restrict__ part) {
  __shared__ float4 red[FF_WARPS - 1][8][32];
  const int g = blockIdx.x, split = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n0 = g * G;
  const int k0 = split * KCHUNK + warp * FF_ROWS;
  bool live[GM];
  int any = 0;
#pragma unroll
  for (int b = 0; b < GM; ++b) {
    live[b] = b < G && n0 + b < N && slot_row[n0 + b] >= 0;
    any |= live[b];
  }
  if (!any) return;
  const float* dc = delta ? delta + (int64_t)g * ld : nullptr;
  float4 acc[GM];
#pragma unroll
  for (int b = 0; b < GM; ++b) acc[b] = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4* th4 = reinterpret_cast<const float4*>(theta + O_F1 + (int64_t)k0 * HID) + lane;
  const float4* dl4 = dc ? reinterpret_cast<const float4*>(dc + O_F1 + (int64_t)k0 * HID) + lane : nullptr;
  for (int r0 = 0; r0 < FF_ROWS; r0 += 32) {
    float pv[GM];  // lane l holds the activations of row r0 + l
#pragma unroll
    for (int b = 0; b < GM; ++b)
      pv[b] = live[b] ? __ldg(pooled + (int64_t)(n0 + b) * FLAT + k0 + r0 + lane) : 0.f;
#pragma unroll 4
    for (int r = 0; r < 32; ++r) {
      const int64_t k = r0 + r;
      float4 w = __ldg(th4 + k * (HID / 4));
      if (dl4) {
        const float4 d = __ldcs(dl4 + k * (HID / 4));
        w.x -= d.x; w.y -= d.y; w.z -= d.z; w.w -= d.w;
      }
#pragma unroll
      for (int b = 0; b < GM; ++b) {
        const float p = __shfl_sync(0xffffffffu, pv[b], r);
        acc[b].x = fmaf(p, w.x, acc[b].x);
        acc[b].y = fmaf(p, w.y, acc[b].y);
        acc[b].z = fmaf(p, w.z, acc[b].z);
        acc[b].w = fmaf(p, w.w, acc[b].w);
      }
    }
  }
#pragma unroll
  for (int b0 = 0; b0 < GM; b0 += 8) {
    if (warp > 0) {
#pragma unroll
      for (int b = b0; b < b0 + 8 && b < GM; ++b) red[warp - 1][b - b0][lane] = acc[b];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int b = b0; b < b0 + 8 && b < GM; ++b) {
        float4 a = acc[b];
#pragma unroll
        for (int w = 0; w < FF_WARPS - 1; ++w) {
          const float4 o = red[w][b - b0][lane];
          a.x += o.x; a.y += o.y; a.z += o.z; a.w += o.w;
        }
        if (b < G && n0 + b < N) reinterpret_cast<float4*>(part + ((int64_t)split * N + n0 + b) * HID)[lane] = a;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ head
// one CTA per group.  Eval: per-slot loss / hit.  Train: softmax-CE grad of
// the mean batch loss, dz3, and the fc2 + fc1-bias updates of the client.
__global__ void __launch_bounds__(HID) head_kernel(const float* __restrict__ part,
                                                   const int64_t* __restrict__ slot_row, int N, int G,
                                                   const int32_t* __restrict__ yl,
                                                   const float* __restrict__ theta, float* __restrict__ delta,
                                                   int64_t ld, const int32_t* __restrict__ client_nb, Step st,
                                                   float* __restrict__ dz3, double* __restrict__ slot_loss,
                                                   int32_t* __restrict__ slot_hit, Hist hs, int nsplit,
                                                   __half* __restrict__ dzfh, __half* __restrict__ dzfl,
                                                   float* __restrict__ dzsc) {
  __shared__ float z3[GMAX][HID];
  __shared__ float dzs[GMAX][HID];
  __shared__ float lg[GMAX][NCLS];
  __shared__ float w2[HID * NCLS + NCLS];
  __shared__ int lab[GMAX];
  const int g = blockIdx.x, j = threadIdx.x;
  const int n0 = g * G;
  const bool train = delta != nullptr;
  float* dc = train ? delta + (int64_t)g * ld : nullptr;
  const int nb = train ? client_nb[g] : 0;
  if (train && nb == 0) return;
  for (int i = j; i < HID * NCLS + NCLS; i += blockDim.x) w2[i] = wt(theta, dc, O_F2 + i);
  const float bf1 = wt(theta, dc, O_BF1 + j);
  // factored fc1: z3[b] -= delta_s p_b = sum_{sp < s, bp} coef_sp dz3_{sp,bp} (p_{sp,bp} . p_b):
  // each history dz3 value is loaded once and applied to every new row b (Gram rows in smem)
  float corr[GMAX];
#pragma unroll
  for (int b = 0; b < GMAX; ++b) corr[b] = 0.f;
  if (train && hs.phist && hs.s > 0) {
    __shared__ float gsm[GMAX][FC_RMAX];
    const int Jp = hs.s * G;
    for (int i = j; i < nb * Jp; i += blockDim.x) {
      const int b = i / Jp, r = i - b * Jp;
      gsm[b][r] = hs.gram[((int64_t)g * hs.R + hs.s * G + b) * hs.R + r];
    }
    __syncthreads();
    for (int sp = 0; sp < hs.s; ++sp) {
      const int nbp = hs.nbh[sp * hs.cstride + g];
      const float cf = hist_coef(st.lr, st.mu, hs.s, sp);
      const float* dzp = hs.dz3h + sp * hs.dstride + (int64_t)n0 * HID + j;
      for (int bp = 0; bp < nbp; ++bp) {
        const float d = cf * dzp[bp * HID];
#pragma unroll
        for (int b = 0; b < GMAX; ++b)
          if (b < nb) corr[b] = fmaf(d, gsm[b][sp * G + bp], corr[b]);
      }
    }
  }
  // the K-split partials of two rows at a time: 14 loads in flight, each row summed in split
  // order (bf1 first) -- the same additions as one row at a time
#pragma unroll
  for (int b = 0; b < GMAX; b += 2) {
    if (b >= G) break;
    const int na = n0 + b, nb2 = n0 + b + 1;
    const bool va = na < N && slot_row[na] >= 0;
    const bool vb = b + 1 < G && nb2 < N && slot_row[nb2] >= 0;
    float za = va ? bf1 : 0.f, zb = vb ? bf1 : 0.f;
    int s = 0;
    for (; s + 7 <= nsplit; s += 7) {
      float v[7], w[7];
#pragma unroll
      for (int u = 0; u < 7; ++u) {
        v[u] = va ? part[((int64_t)(s + u) * N + na) * HID + j] : 0.f;
        w[u] = vb ? part[((int64_t)(s + u) * N + nb2) * HID + j] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 7; ++u) {
        za += v[u];
        zb += w[u];
      }
    }
    for (; s < nsplit; ++s) {
      if (va) za += part[((int64_t)s * N + na) * HID + j];
      if (vb) zb += part[((int64_t)s * N + nb2) * HID + j];
    }
    z3[b][j] = za - corr[b];
    if (b + 1 < G) z3[b + 1][j] = zb - corr[b + 1];
  }
  if (j < G) {
    const int n = n0 + j;
    lab[j] = (n < N && slot_row[n] >= 0) ? yl[slot_row[n]] : -1;
  }
  __syncthreads();
  for (int t = j; t < G * NCLS; t += blockDim.x) {
    const int b = t / NCLS, q = t - b * NCLS;
    float v = w2[HID * NCLS + q];
    for (int h = 0; h < HID; ++h) v = fmaf(fmaxf(z3[b][h], 0.f), w2[h * NCLS + q], v);
    lg[b][q] = v;
  }
  __syncthreads();
  if (j < G && lab[j] >= 0) {
    float* row = lg[j];
    float mx = row[0];
    int arg = 0;
    for (int q = 1; q < NCLS; ++q)
      if (row[q] > mx) { mx = row[q]; arg = q; }
    float s = 0.f;
    for (int q = 0; q < NCLS; ++q) s += expf(row[q] - mx);
    if (slot_loss) {  // evaluation, or the first local step (its forward is the eval at theta_t)
      slot_loss[n0 + j] = -((double)row[lab[j]] - (double)mx - (double)logf(s));
      slot_hit[n0 + j] = arg == lab[j];
    }
    if (train) {
      for (int q = 0; q < NCLS; ++q) {
        float p = expf(row[q] - mx) / s;
        if (q == lab[j]) p -= 1.f;
        row[q] = p / (float)nb;
      }
    }
  }
  if (!train) return;
  __syncthreads();
  // dz3 (old fc2 weights), fc1 bias grad
  float gb = 0.f;
  for (int b = 0; b < nb; ++b) {
    float d = 0.f;
#pragma unroll
    for (int q = 0; q < NCLS; ++q) d = fmaf(lg[b][q], w2[j * NCLS + q], d);
    d = z3[b][j] > 0.f ? d : 0.f;
    dz3[(int64_t)(n0 + b) * HID + j] = d;
    dzs[b][j] = d;
    gb += d;
  }
  for (int b = nb; b < G; ++b) dz3[(int64_t)(n0 + b) * HID + j] = 0.f;
  if (dzfh) {
    // scaled fp16 hi / lo of dz3 (A operand of the tcgen05 fc1 backward)
    __shared__ float red[GMAX][HID / 32];
    for (int b = 0; b < nb; ++b) {
      const float m = warp_max(fabsf(dzs[b][j]));
      if ((j & 31) == 0) red[b][j >> 5] = m;
    }
    __syncthreads();
    for (int b = 0; b < nb; ++b) {
      float m = 0.f;
#pragma unroll
      for (int w = 0; w < HID / 32; ++w) m = fmaxf(m, red[b][w]);
      const float sc = m > 0.f ? exp2f(14.f - ceilf(log2f(m))) : 1.f;
      if (j == 0) dzsc[n0 + b] = sc;
      __half h, l;
      split_f16(dzs[b][j] * sc, h, l);
      dzfh[(int64_t)(n0 + b) * HID + j] = h;
      dzfl[(int64_t)(n0 + b) * HID + j] = l;
    }
  }
  if (hs.phist) {
    // coefficients of the history rows in this step's dp: a[b][j] = coef * (dz3_j . dz3_b)
    __syncthreads();
    const int J = hs.s * G;
    float* ac = hs.acoef + (int64_t)g * GMAX * FC_RMAX;
    for (int pr = j; pr < nb * J; pr += blockDim.x) {
      const int b = pr / J, jj = pr - b * J, sp = jj / G, bp = jj - sp * G;
      float a = 0.f;
      if (bp < hs.nbh[sp * hs.cstride + g]) {
        const float* zp = hs.dz3h + sp * hs.dstride + (int64_t)(n0 + bp) * HID;
        for (int h = 0; h < HID; ++h) a = fmaf(dzs[b][h], zp[h], a);
        a *= hist_coef(st.lr, st.mu, hs.s, sp);
      }
      ac[b * FC_RMAX + jj] = a;
    }
  }
  // updates: theta <- theta - lr*(g + mu*(theta - theta_t)) == delta += lr*(g - mu*delta)
  {
    float& dl = dc[O_BF1 + j];
    dl += st.lr * (gb - st.mu * dl);
  }
  for (int t = j; t < HID * NCLS; t += blockDim.x) {
    const int h = t / NCLS, q = t - h * NCLS;
    float gw = 0.f;
    for (int b = 0; b < nb; ++b) gw = fmaf(fmaxf(z3[b][h], 0.f), lg[b][q], gw);
    float& dl = dc[O_F2 + t];
    dl += st.lr * (gw - st.mu * dl);
  }
  if (j < NCLS) {
    float gw = 0.f;
    for (int b = 0; b < nb; ++b) gw += lg[b][j];
    float& dl = dc[O_BF2 + j];
    dl += st.lr * (gw - st.mu * dl);
  }
}

// ------------------------------------------------------- fc1 bwd + update
// grid (C, KSPLIT), 4 warps per CTA, each warp streaming 112 weight rows of
// the client.  Per row: theta_t and delta as float4 per lane (coalesced), the
// gradient p^T dz3 for the lane's 4 units (activations broadcast by shuffles,
// dz3 in registers), delta += lr*(g - mu*delta) written back in the same
// pass; the OLD weights go to a per-warp 16-row smem tile from which each lane
// then computes dp = dz3 W^T for one row (conflict-free padded rows).
constexpr int FB_WARPS = 4, FB_TR = 16, FB_LDW = HID + 1;
constexpr int FC1B_SMEM = (FB_WARPS * FB_TR * FB_LDW + GMAX * HID) * 4;

template <int GM>
__global__ void __launch_bounds__(FB_WARPS * 32) fc1_bwd_kernel(const float* __restrict__ pooled,
                                                                 const float* __restrict__ dz3, int B,
                                                                 const int32_t* __restrict__ client_nb,
                                                                 const float* __restrict__ theta,
                                                                 float* __restrict__ delta, int64_t ld, Step st,
                                                                 float* __restrict__ dp, int rsplit) {
  extern __shared__ float bsm[];
  // grid.y = KSPLIT * rsplit (rsplit 1 or 7): rows are independent, so a few active
  // clients (ragged cohorts) spread their rows over 7x more CTAs
  const int c = blockIdx.x, split = blockIdx.y / rsplit, sub = blockIdx.y - split * rsplit;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = client_nb[c];
  if (nb == 0) return;
  float* dz = bsm;                                     // [GM][HID]
  float* wt_ = bsm + GMAX * HID + warp * FB_TR * FB_LDW;  // this warp's [FB_TR][FB_LDW]
  const int n0 = c * B;
  for (int i = threadIdx.x; i < GM * HID; i += blockDim.x) dz[i] = i < nb * HID ? dz3[(int64_t)n0 * HID + i] : 0.f;
  __syncthreads();
  float4 dzr[GM];
#pragma unroll
  for (int b = 0; b < GM; ++b) dzr[b] = reinterpret_cast<const float4*>(dz + b * HID)[lane];
  float* dc = delta + (int64_t)c * ld;
  const float lr = st.lr, mu = st.mu;
  constexpr int ROWS_PER_WARP = KCHUNK / FB_WARPS;  // 112
  const int rows = ROWS_PER_WARP / rsplit;
  const int kw = split * KCHUNK + warp * ROWS_PER_WARP + sub * rows;
  for (int r0 = 0; r0 < rows; r0 += FB_TR) {
    float pv[GM];  // lane l < FB_TR holds the activations of row r0 + l
#pragma unroll
    for (int b = 0; b < GM; ++b)
      pv[b] = (b < nb && lane < FB_TR) ? __ldg(pooled + (int64_t)(n0 + b) * FLAT + kw + r0 + lane) : 0.f;
#pragma unroll 4
    for (int r = 0; r < FB_TR; ++r) {
      const int64_t off = O_F1 + (int64_t)(kw + r0 + r) * HID;
      const float4 th = __ldg(reinterpret_cast<const float4*>(theta + off) + lane);
      float4* dptr = reinterpret_cast<float4*>(dc + off) + lane;
      const float4 d = *dptr;
      float* wrow = wt_ + r * FB_LDW + 4 * lane;
      wrow[0] = th.x - d.x; wrow[1] = th.y - d.y; wrow[2] = th.z - d.z; wrow[3] = th.w - d.w;
      float4 gw = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int b = 0; b < GM; ++b) {
        const float p = __shfl_sync(0xffffffffu, pv[b], r);
        gw.x = fmaf(p, dzr[b].x, gw.x);
        gw.y = fmaf(p, dzr[b].y, gw.y);
        gw.z = fmaf(p, dzr[b].z, gw.z);
        gw.w = fmaf(p, dzr[b].w, gw.w);
      }
      *dptr = make_float4(d.x + lr * (gw.x - mu * d.x), d.y + lr * (gw.y - mu * d.y),
                          d.z + lr * (gw.z - mu * d.z), d.w + lr * (gw.w - mu * d.w));
    }
    __syncwarp();
    // dp[b][row] = sum_j dz[b][j] * w_old[row][j]: lanes 0..15 take one row each for b even,
    // lanes 16..31 for b odd (two samples in flight per row)
    {
      const int r = lane & (FB_TR - 1), bpar = lane >> 4;
      const float* wr = wt_ + r * FB_LDW;
      for (int b = bpar; b < nb; b += 2) {
        const float* zb = dz + b * HID;
        float s0 = 0.f, s1 = 0.f;
#pragma unroll 8
        for (int j = 0; j < HID; j += 2) {
          s0 = fmaf(zb[j], wr[j], s0);
          s1 = fmaf(zb[j + 1], wr[j + 1], s1);
        }
        dp[(int64_t)(n0 + b) * FLAT + kw + r0 + r] = s0 + s1;
      }
    }
    __syncwarp();
  }
}

// --------------------------------------------- conv2 backward (data) -> dz1
// one CTA per active slot; g = dp * relu'(at argmax) kept sparse with its
// window code; thread per a1 position, 32 input-channel accumulators
constexpr int C2X_SMEM = (9 * C2 * C1 + C2 * NPOOL) * 4 + C2 * NPOOL;

__global__ void __launch_bounds__(256) conv2_bwd_x_kernel(const float* __restrict__ dp,
                                                          const float* __restrict__ pooled,
                                                          const uint8_t* __restrict__ code,
                                                          const float* __restrict__ a1,  // hi part: sign of a1
                                                          const int64_t* __restrict__ slot_row, int B,
                                                          const float* __restrict__ theta,
                                                          const float* __restrict__ delta, int64_t ld,
                                                          float* __restrict__ dz1) {
  extern __shared__ float sm[];
  float* ws = sm;                      // [tap9][o64][ci32]
  float* gs = ws + 9 * C2 * C1;        // [o64][196]
  uint8_t* cs = reinterpret_cast<uint8_t*>(gs + C2 * NPOOL);
  const int n = blockIdx.x;
  if (slot_row[n] < 0) return;
  const float* dc = delta + (int64_t)(n / B) * ld;
  for (int i = threadIdx.x; i < C2 * C1 * 9; i += blockDim.x) {
    const int o = i / (C1 * 9), r = i - o * (C1 * 9), ci = r / 9, tap = r - ci * 9;
    ws[(tap * C2 + o) * C1 + ci] = theta[O_W2 + i] - dc[O_W2 + i];
  }
  for (int i = threadIdx.x; i < FLAT; i += blockDim.x) {
    const int64_t s = (int64_t)n * FLAT + i;
    gs[i] = pooled[s] > 0.f ? dp[s] : 0.f;
    cs[i] = code[s];
  }
  __syncthreads();
  const float* a1n = a1 + (int64_t)n * A1;
  float* out = dz1 + (int64_t)n * A1;
  for (int p = threadIdx.x; p < S1 * S1; p += blockDim.x) {
    const int y = p / S1, x = p - y * S1;
    float acc[C1];
#pragma unroll
    for (int ci = 0; ci < C1; ++ci) acc[ci] = 0.f;
#pragma unroll 1
    for (int tap = 0; tap < 9; ++tap) {
      const int ky = tap / 3, kx = tap - ky * 3;
      const int zy = y - ky, zx = x - kx;
      if (zy < 0 || zx < 0 || zy >= S2 || zx >= S2) continue;
      const int pp = (zy >> 1) * SP + (zx >> 1);
      const int sub = ((zy & 1) << 1) | (zx & 1);
      const float* wr = ws + tap * C2 * C1;
#pragma unroll 2
      for (int o = 0; o < C2; ++o) {
        const float gv = cs[o * NPOOL + pp] == sub ? gs[o * NPOOL + pp] : 0.f;
        if (gv == 0.f) continue;
        const float4* w4 = reinterpret_cast<const float4*>(wr + o * C1);
#pragma unroll
        for (int q = 0; q < C1 / 4; ++q) {
          const float4 wv = w4[q];
          acc[4 * q] = fmaf(gv, wv.x, acc[4 * q]);
          acc[4 * q + 1] = fmaf(gv, wv.y, acc[4 * q + 1]);
          acc[4 * q + 2] = fmaf(gv, wv.z, acc[4 * q + 2]);
          acc[4 * q + 3] = fmaf(gv, wv.w, acc[4 * q + 3]);
        }
      }
    }
    const float4* am = reinterpret_cast<const float4*>(a1n + (int64_t)p * C1);
    float4* dst = reinterpret_cast<float4*>(out + (int64_t)p * C1);
#pragma unroll
    for (int q = 0; q < C1 / 4; ++q) {
      const float4 m = am[q];
      dst[q] = make_float4(m.x > 0.f ? acc[4 * q] : 0.f, m.y > 0.f ? acc[4 * q + 1] : 0.f,
                           m.z > 0.f ? acc[4 * q + 2] : 0.f, m.w > 0.f ? acc[4 * q + 3] : 0.f);
    }
  }
}

// ------------------------------------------- conv2 backward (weights) + update
// one CTA per client: dW2[o][tap][ci] = sum over slots and pooled positions
// of g * a1(window argmax + tap); thread = (o, quarter of the 288 (tap,ci))
constexpr int C2W_SMEM = (S1 * S1 * A1P + C2 * NPOOL) * 4 + C2 * NPOOL;

__global__ void __launch_bounds__(256) conv2_bwd_w_kernel(const float* __restrict__ dp,
                                                          const float* __restrict__ pooled,
                                                          const uint8_t* __restrict__ code,
                                                          const float* __restrict__ a1h,
                                                          const float* __restrict__ a1l, int B,
                                                          const int32_t* __restrict__ client_nb,
                                                          float* __restrict__ delta, int64_t ld, Step st) {
  extern __shared__ float sm[];
  float* as = sm;                      // [900][33]
  float* gs = as + S1 * S1 * A1P;      // [64][196]
  uint8_t* cs = reinterpret_cast<uint8_t*>(gs + C2 * NPOOL);
  const int c = blockIdx.x;
  const int nb = client_nb[c];
  if (nb == 0) return;
  const int o = threadIdx.x >> 2, quarter = threadIdx.x & 3;  // 72 (tap,ci) per thread
  float acc[72];
#pragma unroll
  for (int i = 0; i < 72; ++i) acc[i] = 0.f;
  float gbias = 0.f;
  for (int b = 0; b < nb; ++b) {
    const int64_t n = (int64_t)c * B + b;
    __syncthreads();
    for (int i = threadIdx.x; i < A1; i += blockDim.x)
      as[(i >> 5) * A1P + (i & 31)] = a1h[n * A1 + i] + (a1l ? a1l[n * A1 + i] : 0.f);
    for (int i = threadIdx.x; i < FLAT; i += blockDim.x) {
      gs[i] = pooled[n * FLAT + i] > 0.f ? dp[n * FLAT + i] : 0.f;
      cs[i] = code[n * FLAT + i];
    }
    __syncthreads();
    for (int pp = 0; pp < NPOOL; ++pp) {
      const float gv = gs[o * NPOOL + pp];
      if (gv == 0.f) continue;
      gbias += gv;
      const int sub = cs[o * NPOOL + pp];
      const int y = 2 * (pp / SP) + (sub >> 1), x = 2 * (pp % SP) + (sub & 1);
#pragma unroll
      for (int i = 0; i < 72; ++i) {
        const int k = quarter * 72 + i, tap = k >> 5, ci = k & 31;
        const int ky = tap / 3, kx = tap - ky * 3;
        acc[i] = fmaf(gv, as[((y + ky) * S1 + x + kx) * A1P + ci], acc[i]);
      }
    }
  }
  float* dc = delta + (int64_t)c * ld;
#pragma unroll
  for (int i = 0; i < 72; ++i) {
    const int k = quarter * 72 + i, tap = k >> 5, ci = k & 31;
    float& dl = dc[O_W2 + (int64_t)o * C1 * 9 + ci * 9 + tap];
    dl += st.lr * (acc[i] - st.mu * dl);
  }
  // bias: the four threads of channel o hold identical sums; one writes
  if (quarter == 0) {
    float& dl = dc[O_B2 + o];
    dl += st.lr * (gbias - st.mu * dl);
  }
}

// ------------------------------------------- conv1 backward (weights) + update
// one CTA per client, 12 warps: warp = (8 output channels, 1 input channel) tile
// holding the 8 x 9 taps of dW1 in registers; lanes stride over the 900
// positions of each of the client's samples (dz1 rows read straight from HBM,
// the 3x32x32 input from smem); lane partials are warp-reduced at the end.
constexpr int C1B_WARPS = 12;

__global__ void __launch_bounds__(C1B_WARPS * 32) conv1_bwd_w_kernel(const float* __restrict__ X,
                                                                    const int64_t* __restrict__ slot_row,
                                                                    const float* __restrict__ dz1, int B,
                                                                    const int32_t* __restrict__ client_nb,
                                                                    float* __restrict__ delta, int64_t ld, Step st) {
  __shared__ float img[IMG];
  const int c = blockIdx.x;
  const int nb = client_nb[c];
  if (nb == 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int og = warp & 3, ci = warp >> 2;  // channels 8*og .. 8*og+7, input channel ci
  float acc[8][9], accb[8];
#pragma unroll
  for (int o = 0; o < 8; ++o) {
    accb[o] = 0.f;
#pragma unroll
    for (int t = 0; t < 9; ++t) acc[o][t] = 0.f;
  }
  for (int b = 0; b < nb; ++b) {
    const int64_t n = (int64_t)c * B + b;
    const int64_t row = slot_row[n];
    __syncthreads();
    for (int i = threadIdx.x; i < IMG; i += blockDim.x) img[i] = X[row * IMG + i];
    __syncthreads();
    const float* dzn = dz1 + n * A1 + og * 8;
    const float* im = img + ci * S0 * S0;
    for (int p = lane; p < S1 * S1; p += 32) {
      const int y = p / S1, x = p - y * S1;
      const float4 d0 = __ldg(reinterpret_cast<const float4*>(dzn + (int64_t)p * C1));
      const float4 d1 = __ldg(reinterpret_cast<const float4*>(dzn + (int64_t)p * C1) + 1);
      const float dv[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
      float pv[9];
#pragma unroll
      for (int t = 0; t < 9; ++t) pv[t] = im[(y + t / 3) * S0 + x + t % 3];
#pragma unroll
      for (int o = 0; o < 8; ++o) {
        accb[o] += dv[o];
#pragma unroll
        for (int t = 0; t < 9; ++t) acc[o][t] = fmaf(dv[o], pv[t], acc[o][t]);
      }
    }
  }
  float* dc = delta + (int64_t)c * ld;
#pragma unroll
  for (int o = 0; o < 8; ++o) {
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      const float g = warp_sum(acc[o][t]);
      if (lane == 0) {
        float& dl = dc[O_W1 + (int64_t)(og * 8 + o) * (C0 * 9) + ci * 9 + t];
        dl += st.lr * (g - st.mu * dl);
      }
    }
    if (ci == 0) {
      const float gb = warp_sum(accb[o]);
      if (lane == 0) {
        float& dl = dc[O_B1 + og * 8 + o];
        dl += st.lr * (gb - st.mu * dl);
      }
    }
  }
}

__global__ void eval_reduce_kernel(const double* __restrict__ slot_loss, const int32_t* __restrict__ slot_hit,
                                   const int32_t* __restrict__ slot_client, int N, int64_t r0,
                                   const int64_t* __restrict__ prefix, int C, double* __restrict__ loss_sum,
                                   int32_t* __restrict__ correct) {
  // clients overlapping the chunk [r0, r0+N): sum their slots in row order
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int64_t lo = max(prefix[c], r0), hi = min(prefix[c + 1], r0 + N);
  if (lo >= hi) return;
  double s = 0.0;
  int h = 0;
  for (int64_t r = lo; r < hi; ++r) {
    s += slot_loss[r - r0];
    h += slot_hit[r - r0];
  }
  loss_sum[c] += s;
  correct[c] += h;
}

// zero every client's delta row except [skip0, skip1) (float4; ld, skip0, skip1 multiples of 4)
// zero every client row except the columns [skip0, skip1) (the factored fc1 block, written whole
// later): the grid strides over the kept quads only (skip0 / skip1 multiples of 4)
__global__ void zero_delta_kernel(float* __restrict__ delta, int64_t ld, int C, int64_t skip0, int64_t skip1) {
  const int64_t q = ld >> 2, q0 = skip0 >> 2, qs = (skip1 - skip0) >> 2, kept = q - qs;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)C * kept;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / kept, j = i - c * kept;
    reinterpret_cast<float4*>(delta)[c * q + (j < q0 ? j : j + qs)] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// ------------------------------------------------------ fc1 in factored form
// fc1's SGD update of one step is the rank-nb outer product dz3^T P of the
// step's batch, so within one local-training run client c's fc1 weights are
//   W_s = theta_t - delta_s,  delta_s = sum_{s' < s} lr (1 - lr mu)^{s-1-s'} dz3_{s'}^T P_{s'}
// (exactly the recursion delta += lr*(g - mu*delta) of the dense path).  With
// at most FC_RMAX history rows per client the run never forms delta_s:
//   z3 = theta_t p - sum_j coef_j dz3_j (p_j . p)      (fc1_fwd at theta_t + Gram + head)
//   dp = theta_t dz3 - sum_j coef_j (dz3_j . dz3) p_j  (fc1_bwd_fact)
// and the client's fc1 delta is written once at the end (fc1_materialize).
// Per step that replaces the 6.4 MB read (forward) + 12.8 MB read/write
// (backward) of every client's fc1 delta with the history rows (~0.5 MB per
// earlier step) and the L2-resident theta_t.

// Gram rows of the current step: gram[c][(s*B + b)][j] = p_{s,b} . p_j for j < (s+1)*B.
// One CTA per client; 64-wide K chunks of all (s+1)*B rows staged in smem;
// thread = 2 current rows x 4 history rows, float4 along K.
constexpr int GR_KC = 64, GR_KP = GR_KC + 4;
__global__ void __launch_bounds__(128) fc1_gram_kernel(Hist hs, int B) {
  __shared__ __align__(16) float tile[FC_RMAX][GR_KP];
  const int c = blockIdx.x, t = threadIdx.x;
  const int s = hs.s, J = (s + 1) * B;
  if (hs.nbh[s * hs.cstride + c] == 0) return;
  const int jq = t & 15, bq = t >> 4;
  const int rb0 = min(s * B + bq, FC_RMAX - 1), rb1 = min(s * B + bq + 8, FC_RMAX - 1);
  double acc[2][4] = {};  // per-chunk fp32 partials summed in fp64: the Gram entries are
                          // long (12544-term) sums of positive products
  for (int k0 = 0; k0 < FLAT; k0 += GR_KC) {
    for (int i = t; i < J * (GR_KC / 4); i += blockDim.x) {
      const int row = i >> 4, c4 = i & 15, sp = row / B, bp = row - sp * B;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (bp < hs.nbh[sp * hs.cstride + c])
        v = __ldg(reinterpret_cast<const float4*>(hs.phist + sp * hs.pstride + (int64_t)(c * B + bp) * FLAT + k0) + c4);
      *reinterpret_cast<float4*>(&tile[row][4 * c4]) = v;
    }
    __syncthreads();
    float part[2][4] = {};
#pragma unroll 4
    for (int kk = 0; kk < GR_KC; kk += 4) {
      const float4 x0 = *reinterpret_cast<const float4*>(&tile[rb0][kk]);
      const float4 x1 = *reinterpret_cast<const float4*>(&tile[rb1][kk]);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 y = *reinterpret_cast<const float4*>(&tile[jq + 16 * i][kk]);
        part[0][i] = fmaf(x0.x, y.x, fmaf(x0.y, y.y, fmaf(x0.z, y.z, fmaf(x0.w, y.w, part[0][i]))));
        part[1][i] = fmaf(x1.x, y.x, fmaf(x1.y, y.y, fmaf(x1.z, y.z, fmaf(x1.w, y.w, part[1][i]))));
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc[0][i] += part[0][i];
      acc[1][i] += part[1][i];
    }
    __syncthreads();
  }
  float* gr = hs.gram + (int64_t)c * hs.R * hs.R;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int b = bq + 8 * u;
    if (b >= B) continue;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j = jq + 16 * i;
      if (j < J) gr[(s * B + b) * hs.R + j] = (float)acc[u][i];
    }
  }
}

// Split-K Gram for the current step: grid (4, nks, C), CTA = 2 warps, warp owns
// history rows j = 16 z + 8 w .. +7, lane = 4 consecutive k (float4, strided by 128
// over the CTA's K range): per k-quad the lane loads the step's nb <= GM new rows and
// its 8 history rows (coalesced 512-byte warp loads, 18 in flight per warp) and does
// GM x 8 x 4 FMAs; each lane sums <= 98 products per (b, j) in fp32 (pooled >= 0: no
// cancellation), the warp tree-reduces and the K splits are summed in fp64 in fixed
// order by fc1_gram_reduce_kernel.  Small CTAs so that the register file, not
// exited warps, bounds residency (the old 8-warp CTA left 15% of warps active).
constexpr int GR_KS = 14;                      // max K splits per client (runtime: gridDim.y = 7 or 14)
constexpr int GR_JW = 8;                       // history rows per warp
constexpr int GR_WARPS = 2;                    // warps per CTA
constexpr int GR_Z = FC_RMAX / (GR_JW * GR_WARPS);  // 4 row groups
static_assert(FLAT % (GR_KS * 128) == 0 && FLAT % (7 * 128) == 0, "gram K split");
template <int GM>
__global__ void __launch_bounds__(GR_WARPS * 32) fc1_gram_split_kernel(Hist hs, int B, double* __restrict__ part) {
  // grid (row groups, K splits, clients): the row-group CTAs of one (client, K split) read
  // the same new rows and run back to back, so the rereads hit L2 (client-fastest order sent
  // them to DRAM: a row group's pass over all clients is ~500 MB)
  const int c = blockIdx.z, ks = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = hs.s, J = (s + 1) * B;
  const int nb = hs.nbh[s * hs.cstride + c];
  const int j0 = (blockIdx.x * GR_WARPS + warp) * GR_JW;
  if (nb == 0 || j0 >= J) return;
  // new rows are consecutive slots of step s; history rows as 32-bit element offsets
  // (the host checks S * N * FLAT < 2^31)
  const float* newp = hs.phist + s * hs.pstride + (int64_t)c * B * FLAT;
  uint32_t hoff[GR_JW];
  int live = 0;
#pragma unroll
  for (int i = 0; i < GR_JW; ++i) {
    const int j = min(j0 + i, J - 1), sp = j / B, bp = j - sp * B;
    const bool act = j0 + i < J && bp < hs.nbh[sp * hs.cstride + c];
    live |= act << i;
    hoff[i] = (uint32_t)(sp * hs.pstride + (int64_t)(c * B + bp) * FLAT);
  }
  float acc[GM][GR_JW];
#pragma unroll
  for (int b = 0; b < GM; ++b)
#pragma unroll
    for (int i = 0; i < GR_JW; ++i) acc[b][i] = 0.f;
  const int nks = gridDim.y;
  const int k0 = ks * (FLAT / nks), k1 = k0 + FLAT / nks;
#pragma unroll 1
  for (int k = k0 + 4 * lane; k < k1; k += 128) {
    float4 x[GM], h[GR_JW];
#pragma unroll
    for (int b = 0; b < GM; ++b)
      x[b] = b < nb ? __ldg(reinterpret_cast<const float4*>(newp + b * FLAT + k)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int i = 0; i < GR_JW; ++i) h[i] = __ldg(reinterpret_cast<const float4*>(hs.phist + hoff[i] + k));
#pragma unroll
    for (int b = 0; b < GM; ++b)
#pragma unroll
      for (int i = 0; i < GR_JW; ++i)
        acc[b][i] = fmaf(x[b].w, h[i].w, fmaf(x[b].z, h[i].z, fmaf(x[b].y, h[i].y, fmaf(x[b].x, h[i].x, acc[b][i]))));
  }
  double* out = part + (((int64_t)c * nks + ks) * GMAX) * FC_RMAX;
#pragma unroll
  for (int b = 0; b < GM; ++b)
#pragma unroll
    for (int i = 0; i < GR_JW; ++i) {
      const float v = warp_sum(acc[b][i]);
      if (lane == 0 && b < nb && ((live >> i) & 1)) out[b * FC_RMAX + j0 + i] = (double)v;
    }
}

__global__ void __launch_bounds__(256) fc1_gram_reduce_kernel(Hist hs, int B, int nks, const double* __restrict__ part) {
  const int c = blockIdx.x;
  const int s = hs.s, J = (s + 1) * B;
  const int nb = hs.nbh[s * hs.cstride + c];
  float* gr = hs.gram + (int64_t)c * hs.R * hs.R;
  for (int i = threadIdx.x; i < nb * J; i += blockDim.x) {
    const int b = i / J, j = i - b * J, sp = j / B, bp = j - sp * B;
    if (bp >= hs.nbh[sp * hs.cstride + c]) continue;
    double v = 0.0;
    for (int ks = 0; ks < nks; ++ks) v += part[(((int64_t)c * nks + ks) * GMAX + b) * FC_RMAX + j];
    gr[(s * B + b) * hs.R + j] = (float)v;
  }
}

// dp = dz3 theta_t^T - sum_j a[b][j] p_j.  grid (C, KSPLIT), 4 warps: the
// theta_t part as in fc1_bwd (warp-streamed 16-row tiles, no delta), staged
// in smem; then thread = 4 consecutive k of the chunk subtracts the history
// rows (coalesced float4 reads) and writes dp.
constexpr int FF_DPB = GMAX * KCHUNK;
constexpr int FC1F_SMEM = (FB_WARPS * FB_TR * FB_LDW + GMAX * HID + GMAX * FC_RMAX + FF_DPB) * 4;

template <int GM>
__global__ void __launch_bounds__(FB_WARPS * 32) fc1_bwd_fact_kernel(const float* __restrict__ dz3, int B,
                                                                      const int32_t* __restrict__ client_nb,
                                                                      const float* __restrict__ theta, Hist hs,
                                                                      float* __restrict__ dp) {
  extern __shared__ float bsm[];
  const int c = blockIdx.x, split = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = client_nb[c];
  if (nb == 0) return;
  float* dz = bsm;                                          // [GMAX][HID]
  float* ac = dz + GMAX * HID;                              // [GMAX][FC_RMAX]
  float* dpb = ac + GMAX * FC_RMAX;                         // [GMAX][KCHUNK]
  float* wt_ = dpb + FF_DPB + warp * FB_TR * FB_LDW;        // this warp's [FB_TR][FB_LDW]
  const int n0 = c * B;
  const int J = hs.s * B;
  for (int i = threadIdx.x; i < GM * HID; i += blockDim.x) dz[i] = i < nb * HID ? dz3[(int64_t)n0 * HID + i] : 0.f;
  for (int i = threadIdx.x; i < nb * J; i += blockDim.x) {
    const int b = i / J, jj = i - b * J;
    ac[b * FC_RMAX + jj] = hs.acoef[((int64_t)c * GMAX + b) * FC_RMAX + jj];
  }
  __syncthreads();
  float4 dzr[GM];
#pragma unroll
  for (int b = 0; b < GM; ++b) dzr[b] = reinterpret_cast<const float4*>(dz + b * HID)[lane];
  (void)dzr;
  constexpr int ROWS_PER_WARP = KCHUNK / FB_WARPS;  // 112
  const int k0 = split * KCHUNK;
  const int kw = warp * ROWS_PER_WARP;
  for (int r0 = 0; r0 < ROWS_PER_WARP; r0 += FB_TR) {
#pragma unroll 4
    for (int r = 0; r < FB_TR; ++r) {
      const int64_t off = O_F1 + (int64_t)(k0 + kw + r0 + r) * HID;
      const float4 th = __ldg(reinterpret_cast<const float4*>(theta + off) + lane);
      float* wrow = wt_ + r * FB_LDW + 4 * lane;
      wrow[0] = th.x; wrow[1] = th.y; wrow[2] = th.z; wrow[3] = th.w;
    }
    __syncwarp();
    {
      const int r = lane & (FB_TR - 1), bpar = lane >> 4;
      const float* wr = wt_ + r * FB_LDW;
      for (int b = bpar; b < nb; b += 2) {
        const float* zb = dz + b * HID;
        float s0 = 0.f, s1 = 0.f;
#pragma unroll 8
        for (int j = 0; j < HID; j += 2) {
          s0 = fmaf(zb[j], wr[j], s0);
          s1 = fmaf(zb[j + 1], wr[j + 1], s1);
        }
        dpb[b * KCHUNK + kw + r0 + r] = s0 + s1;
      }
    }
    __syncwarp();
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t < KCHUNK / 4) {
    float4 acc[GM];
#pragma unroll
    for (int b = 0; b < GM; ++b)
      acc[b] = b < nb ? *reinterpret_cast<const float4*>(dpb + b * KCHUNK + 4 * t) : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int jj = 0; jj < J; ++jj) {
      const int sp = jj / B, bp = jj - sp * B;
      if (bp >= hs.nbh[sp * hs.cstride + c]) continue;
      const float4 p =
          __ldg(reinterpret_cast<const float4*>(hs.phist + sp * hs.pstride + (int64_t)(n0 + bp) * FLAT + k0) + t);
#pragma unroll
      for (int b = 0; b < GM; ++b) {
        const float a = ac[b * FC_RMAX + jj];
        acc[b].x = fmaf(-a, p.x, acc[b].x);
        acc[b].y = fmaf(-a, p.y, acc[b].y);
        acc[b].z = fmaf(-a, p.z, acc[b].z);
        acc[b].w = fmaf(-a, p.w, acc[b].w);
      }
    }
#pragma unroll
    for (int b = 0; b < GM; ++b)
      if (b < nb) reinterpret_cast<float4*>(dp + (int64_t)(n0 + b) * FLAT + k0)[t] = acc[b];
  }
}

// end of the run: delta_fc1[c][k][h] = sum_j coef_j dz3_j[h] p_j[k] over the
// client's S_c active steps.  grid (C, FLAT/128); CTA = 128 k x 128 h, thread
// = 8 k x 8 h register tile over the <= FC_RMAX history rows in smem.
constexpr int FM_K = 128;
constexpr int FC1M_SMEM = 2 * FC_RMAX * 128 * 4;
__global__ void __launch_bounds__(256) fc1_materialize_kernel(Hist hs, int S, int B, float lr, float mu,
                                                              float* __restrict__ delta, int64_t ld) {
  extern __shared__ __align__(16) float msm[];
  float* U = msm;                  // [FC_RMAX][HID]
  float* P = msm + FC_RMAX * HID;  // [FC_RMAX][FM_K]
  const int c = blockIdx.x, k0 = blockIdx.y * FM_K, t = threadIdx.x;
  int Sc = 0;
  while (Sc < S && hs.nbh[Sc * hs.cstride + c] > 0) ++Sc;
  const int J = Sc * B;
  for (int i = t; i < J * (HID / 4); i += blockDim.x) {
    const int j = i / (HID / 4), q = i - j * (HID / 4), sp = j / B, bp = j - sp * B;
    float4 u = make_float4(0.f, 0.f, 0.f, 0.f), p = u;
    if (bp < hs.nbh[sp * hs.cstride + c]) {
      const float cf = hist_coef(lr, mu, Sc, sp);
      u = __ldg(reinterpret_cast<const float4*>(hs.dz3h + sp * hs.dstride + (int64_t)(c * B + bp) * HID) + q);
      u.x *= cf; u.y *= cf; u.z *= cf; u.w *= cf;
      p = __ldg(reinterpret_cast<const float4*>(hs.phist + sp * hs.pstride + (int64_t)(c * B + bp) * FLAT + k0) + q);
    }
    reinterpret_cast<float4*>(U + j * HID)[q] = u;
    reinterpret_cast<float4*>(P + j * FM_K)[q] = p;
  }
  __syncthreads();
  const int hb = t & 15, kb = t >> 4;
  float acc[8][8] = {};
  for (int j = 0; j < J; ++j) {
    const float4 u0 = reinterpret_cast<const float4*>(U + j * HID)[2 * hb];
    const float4 u1 = reinterpret_cast<const float4*>(U + j * HID)[2 * hb + 1];
    const float4 p0 = reinterpret_cast<const float4*>(P + j * FM_K)[2 * kb];
    const float4 p1 = reinterpret_cast<const float4*>(P + j * FM_K)[2 * kb + 1];
    const float uu[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
    const float pp[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 8; ++b) acc[a][b] = fmaf(pp[a], uu[b], acc[a][b]);
  }
  float* out = delta + (int64_t)c * ld + O_F1 + (int64_t)(k0 + 8 * kb) * HID + 8 * hb;
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    reinterpret_cast<float4*>(out + a * HID)[0] = make_float4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]);
    reinterpret_cast<float4*>(out + a * HID)[1] = make_float4(acc[a][4], acc[a][5], acc[a][6], acc[a][7]);
  }
}


// ================================================================ tcgen05
// The three conv2 contractions run on the 5th-generation tensor cores with
// kind::f16 (fp16 inputs, fp32 accumulation in TMEM).  fp32 accuracy comes
// from a 3-term split: every operand x is scaled by a power of two s (per
// sample for activations / gradients, per client for weights) so |x s| <=
// 2^15, then stored as hi = fp16(x s) and lo = fp16(x s - hi); products are
// hi*hi + hi*lo + lo*hi (the dropped lo*lo is ~2^-22 relative).  The hi*hi
// ("main") and cross terms accumulate in separate TMEM accumulators, summed
// with round-to-nearest on the CUDA cores in the epilogue.  TMEM fp32
// accumulation chains of up to 36 K=16 MMAs were measured as accurate as a
// sequential fp32 sum (tools/microbench/acc_bench.cu: mean error 1-3e-8 of sum|p|);
// the conv kernels chain at most 18 (forward / backward-data: 9 taps x K
// steps) or 15 (weight gradient: one 240-position block), longer sums are
// drained into fp32 registers.  Per-client delta error 2-7e-7 relative,
// the same as FP32 FFMA.
constexpr int TC_THREADS = 192;                 // warp 0 TMA, warp 1 TMEM + MMA, warps 2-5 epilogue

// host: driver entry point for cuTensorMapEncodeTiled (cudart is linked statically)
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

int tensor_map_4d_f16(CUtensorMap* map, const __half* base, const cuuint64_t dims[4], const cuuint64_t strides[3],
                      const cuuint32_t box[4], CUtensorMapSwizzle swz) {
  auto fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return FB_ERR_CUDA;
  }
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<__half*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (fp16) failed (%d)", (int)r);
    return FB_ERR_CUDA;
  }
  return FB_OK;
}
// fp16 a1 NHWC [N][30][30][32] as {32, 30, 30, N}; 64-byte swizzle (32 ci x 2 B rows)
int a1f_tensor_map(CUtensorMap* map, const __half* a1, int N, int box_w, int box_h) {
  const cuuint64_t dims[4] = {(cuuint64_t)C1, (cuuint64_t)S1, (cuuint64_t)S1, (cuuint64_t)N};
  const cuuint64_t strides[3] = {(cuuint64_t)C1 * 2, (cuuint64_t)S1 * C1 * 2, (cuuint64_t)S1 * S1 * C1 * 2};
  const cuuint32_t box[4] = {(cuuint32_t)C1, (cuuint32_t)box_w, (cuuint32_t)box_h, 1};
  return tensor_map_4d_f16(map, a1, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_64B);
}
// fp16 dz2 NHWC [N][28][28][64] as {64, 28, 28, N}; 128-byte swizzle (64 o x 2 B rows)
int dzf_tensor_map(CUtensorMap* map, const __half* dz, int N, int box_w, int box_h) {
  const cuuint64_t dims[4] = {(cuuint64_t)C2, (cuuint64_t)S2, (cuuint64_t)S2, (cuuint64_t)N};
  const cuuint64_t strides[3] = {(cuuint64_t)C2 * 2, (cuuint64_t)S2 * C2 * 2, (cuuint64_t)S2 * S2 * C2 * 2};
  const cuuint32_t box[4] = {(cuuint32_t)C2, (cuuint32_t)box_w, (cuuint32_t)box_h, 1};
  return tensor_map_4d_f16(map, dz, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

// offsets of fp16 element (row, k) in K-major swizzled tiles
__host__ __device__ __forceinline__ uint32_t sw64_off16(uint32_t row, uint32_t k) {   // 32 fp16 per 64 B row
  return row * 64u + ((((k >> 3) ^ ((row >> 1) & 3u)) << 4) | ((k & 7u) << 1));
}
__host__ __device__ __forceinline__ uint32_t sw128_off16(uint32_t row, uint32_t k) {  // 64 fp16 per 128 B row
  return row * 128u + ((((k >> 3) ^ (row & 7u)) << 4) | ((k & 7u) << 1));
}
// power-of-two scale putting max |x| at ~2^14 (1 when the block is all zero)
__device__ __forceinline__ float block_scale(float m, float* red) {
  m = warp_max(m);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  float t = (threadIdx.x & 31) < (int)(blockDim.x >> 5) ? red[threadIdx.x & 31] : 0.f;
  t = warp_max(t);
  return t > 0.f ? exp2f(14.f - ceilf(log2f(t))) : 1.f;
}

// ------------------------------------------------- conv2 forward (tcgen05)
// Implicit GEMM per sample: Z[m, o] = sum_{tap, ci} a1[y+ky, x+kx, ci] W[o, ci, ky, kx].
// Output positions run in the 30-wide space of a1 (m = r*30 + x; columns 28,
// 29 are discarded), where the tap shift (ky, kx) is the whole-row offset
// ky*30 + kx.  An M tile = 4 conv rows = 120 rows (the UMMA M = 128 tile's
// last 8 rows are don't-care), N = 64, K = 9 taps x 32 ci.  Per tile ONE
// 4-D TMA box {32 ci, 30 x, 7 y, 1 n} of the NHWC fp16 a1 (hi and lo, rows
// past the image zero-filled) is staged as 64-byte K-major SWIZZLE_64B rows;
// the nine tap operands are the same band with the descriptor start moved by
// (ky*30 + kx) rows (the swizzle is a function of the absolute smem address,
// so a row-shifted start stays a valid canonical tile).  Each a1 byte crosses
// L2 -> SMEM 7/4 times instead of 9.  The client's 9-tap weights (hi + lo,
// 72 KB) stay resident; TMEM accumulators are double-buffered so the
// epilogue (unscale, bias, ReLU, 2x2 max-pool with argmax code) overlaps the
// next tile's MMAs.
constexpr int FW_ROWS = 4;                       // conv rows per M tile
constexpr int FW_MW = FW_ROWS * S1;              // 120 rows in the 30-wide space
constexpr int FW_TILES = S2 / FW_ROWS;           // 7 tiles per sample
constexpr int FW_BAND = FW_ROWS + 3;             // 7 a1 rows per band (6 + the garbage rows' spill)
constexpr int FW_A_TX = FW_BAND * S1 * 64;       // 13440 bytes per TMA box
constexpr int FW_A = 14 * 1024;                  // band part, 1 KB aligned
constexpr int FW_STAGE = 2 * FW_A;               // hi + lo band
constexpr int FW_B_TAP = C2 * 64;                // 4 KB: 64 rows (o) x 32 ci fp16
constexpr int WIMG_BYTES = 9 * 2 * FW_B_TAP;     // 73728: [tap][hi|lo]
constexpr int FW_STAGES = 3;
constexpr int FW_EPI_WARPS = 16;                 // 4 per TMEM lane quadrant, 16 channels each
constexpr int FW_THREADS = (2 + FW_EPI_WARPS) * 32;
constexpr int FW_XLD = 66;                       // x-pooled pairs per channel row (64 + 2: conflict-free)
constexpr int FW_EPI_BYTES = 2 * C2 * FW_XLD * 4; // double-buffered [64 ch][66] x-pooled conv outputs (post-ReLU)
constexpr int FW_SMEM = 1024 + WIMG_BYTES + FW_STAGES * FW_STAGE + FW_EPI_BYTES + 256;
constexpr int FW_ACC = 2 * C2;                   // main | cross accumulators (64 columns each) per tile
constexpr uint32_t FW_IDESC = tc::idesc_f16(128, C2);
constexpr uint32_t FW_IDESC2 = tc::idesc_f16(128, 2 * C2);  // B = [W hi; W lo] stacked along N
static_assert(127 + 2 * S1 + 2 < FW_BAND * S1 && FW_A_TX <= FW_A, "conv2 fwd band: every tap row inside the band");

// per-group conv2 weight image (K-major SWIZZLE_64B: row o, 32 ci), scaled split
// the client's conv2 weights (theta_t - delta_c, or theta_t) as float4 registers:
// 256 threads x WQ quads cover the 18432 weights (O_W2 is 16-byte aligned), all loads
// of a thread in flight together; returns max |w| of the thread's part
constexpr int WQ = C2 * C1 * 9 / 4 / 256;  // 18
static_assert(C2 * C1 * 9 == WQ * 4 * 256 && O_W2 % 4 == 0, "conv2 weight quads");
__device__ __forceinline__ float load_w2(const float* __restrict__ theta, const float* __restrict__ dc,
                                         float4 (&v)[WQ]) {
  const float4* t4 = reinterpret_cast<const float4*>(theta + O_W2);
  const float4* d4 = dc ? reinterpret_cast<const float4*>(dc + O_W2) : nullptr;
  float m = 0.f;
#pragma unroll
  for (int u = 0; u < WQ; ++u) {
    const int q = threadIdx.x + u * 256;
    float4 w = __ldg(t4 + q);
    if (d4) {
      const float4 d = d4[q];
      w.x -= d.x; w.y -= d.y; w.z -= d.z; w.w -= d.w;
    }
    v[u] = w;
    m = fmaxf(m, fmaxf(fmaxf(fabsf(w.x), fabsf(w.y)), fmaxf(fabsf(w.z), fabsf(w.w))));
  }
  return m;
}

__global__ void __launch_bounds__(256) conv2_wimg_kernel(const float* __restrict__ theta,
                                                         const float* __restrict__ delta, int64_t ld,
                                                         const int32_t* __restrict__ client_nb,
                                                         uint8_t* __restrict__ wimg, float* __restrict__ wscale) {
  __shared__ float red[32];
  const int g = blockIdx.x;
  if (delta && client_nb && client_nb[g] == 0) return;
  const float* dc = delta ? delta + (int64_t)g * ld : nullptr;
  float4 v[WQ];
  const float sc = block_scale(load_w2(theta, dc, v), red);
  if (threadIdx.x == 0) wscale[g] = sc;
  // the 72 KB image is assembled in smem (scattered 2-byte swizzled stores) and
  // written out with coalesced 16-byte stores
  extern __shared__ uint4 wim_s[];
  uint8_t* simg = reinterpret_cast<uint8_t*>(wim_s);
#pragma unroll
  for (int u = 0; u < WQ; ++u) {
    const float e4[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = 4 * (threadIdx.x + u * 256) + e;
      const int o = i / (C1 * 9), r = i - o * (C1 * 9), ci = r / 9, tap = r - ci * 9;
      __half h, l;
      split_f16(e4[e] * sc, h, l);
      const uint32_t off = sw64_off16(o, ci);
      *reinterpret_cast<__half*>(simg + (tap * 2 + 0) * FW_B_TAP + off) = h;
      *reinterpret_cast<__half*>(simg + (tap * 2 + 1) * FW_B_TAP + off) = l;
    }
  }
  __syncthreads();
  uint4* img = reinterpret_cast<uint4*>(wimg + (int64_t)g * WIMG_BYTES);
  for (int i = threadIdx.x; i < WIMG_BYTES / 16; i += blockDim.x) img[i] = wim_s[i];
}

#ifdef FB_FWD_PROF
__device__ unsigned long long g_prof[8];
#endif
__global__ void __launch_bounds__(FW_THREADS, 1) conv2_fwd_tc_kernel(
    const __grid_constant__ CUtensorMap tm_hi, const __grid_constant__ CUtensorMap tm_lo,
    const uint8_t* __restrict__ wimg, const float* __restrict__ wscale, int shared_weights,
    const int64_t* __restrict__ slot_row, int N, int G, const float* __restrict__ theta,
    const float* __restrict__ delta, int64_t ld, int B, const float* __restrict__ a1scale,
    float* __restrict__ pooled, uint8_t* __restrict__ code) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = sm;                                        // [9][2][4 KB]
  uint8_t* sA = sB + WIMG_BYTES;                           // [stages][hi 8 KB | lo 8 KB]
  uint8_t* sP = sA + FW_STAGES * FW_STAGE;  // [2][64 ch][128 rows] fp32 conv outputs
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + FW_EPI_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + FW_STAGES;
  uint64_t* tfull = empty + FW_STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);
  __shared__ float bias[C2];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x;
  const int n0 = g * G;
  {  // nothing to do (clients past their last local step, tail of the last chunk): leave before any setup
    // (one slot per thread, one block-wide OR: a serial scan paid an L2 round trip per slot)
    const int b = threadIdx.x;
    if (!__syncthreads_or(b < G && n0 + b < N && slot_row[n0 + b] >= 0)) return;
  }
  const int wg = shared_weights ? 0 : n0 / B;   // weight group (client) of this CTA
  const float* dc = delta ? delta + (int64_t)wg * ld : nullptr;
  if (threadIdx.x < C2) bias[threadIdx.x] = wt(theta, dc, O_B2 + threadIdx.x);
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < FW_STAGES; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], FW_EPI_WARPS);
    }
    tc::mbar_init(bfull, 1);
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc<2 * FW_ACC>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&tm_hi);
      tc::tma_prefetch(&tm_lo);
      tc::mbar_arrive_expect_tx(bfull, WIMG_BYTES);
      tc::bulk_load(sB, wimg + (int64_t)wg * WIMG_BYTES, WIMG_BYTES, bfull);
      int stage = 0;
      uint32_t phase = 0;
      for (int b = 0; b < G; ++b) {
        const int n = n0 + b;
        if (n >= N || slot_row[n] < 0) continue;
        for (int t = 0; t < FW_TILES; ++t) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
#ifdef FB_FWD_NOTMA  // timing experiment only: no operand traffic
          tc::mbar_arrive(&full[stage]);
#else
          tc::mbar_arrive_expect_tx(&full[stage], 2 * FW_A_TX);
          uint8_t* st_ = sA + stage * FW_STAGE;
          tc::tma_load_4d(st_, &tm_hi, 0, 0, FW_ROWS * t, n, &full[stage]);
          tc::tma_load_4d(st_ + FW_A, &tm_lo, 0, 0, FW_ROWS * t, n, &full[stage]);
#endif
          if (++stage == FW_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    tc::mbar_wait(bfull, 0);
    int stage = 0, tile = 0;
    uint32_t phase = 0;
    const uint32_t sA0 = tc::smem_u32(sA), sB0 = tc::smem_u32(sB);
#ifdef FB_FWD_PROF
    long long p_t0 = clock64(), p_te = 0, p_tf = 0;
#endif
    for (int b = 0; b < G; ++b) {
      const int n = n0 + b;
      if (n >= N || slot_row[n] < 0) continue;
      for (int t = 0; t < FW_TILES; ++t, ++tile) {
        const int acc = tile & 1;
#ifdef FB_FWD_PROF
        long long p_a = clock64();
#endif
        tc::mbar_wait(&tempty[acc], ((tile >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem + acc * FW_ACC;
#ifdef FB_FWD_PROF
        long long p_b = clock64();
#endif
        tc::mbar_wait(&full[stage], phase);
        tc::tc_fence_after();
#ifdef FB_FWD_PROF
        long long p_c = clock64();
        p_te += p_b - p_a;
        p_tf += p_c - p_b;
#endif
        if (tc::elect_one()) {
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) {
            const uint32_t ah = sA0 + stage * FW_STAGE + ((tap / 3) * S1 + tap % 3) * 64, al = ah + FW_A;
            const uint32_t bh = sB0 + tap * 2 * FW_B_TAP;  // [hi 64 rows | lo 64 rows]: one 128-row operand
            // K = 32 ci = 2 x 16: the second K step starts 32 B (2 descriptor units) later
            tc::mma2s_f16_ks<2, 2, 2>(d, d + C2, tc::sdesc(ah, 16, 512, 4), tc::sdesc(al, 16, 512, 4),
                                      tc::sdesc(bh, 16, 512, 4), FW_IDESC2, FW_IDESC, tap != 0);
          }
          tc::mma_commit(&empty[stage]);
          tc::mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == FW_STAGES) { stage = 0; phase ^= 1; }
      }
    }
#ifdef FB_FWD_PROF
    if (lane == 0) {
      atomicAdd(&g_prof[0], (unsigned long long)(clock64() - p_t0));
      atomicAdd(&g_prof[1], (unsigned long long)p_te);
      atomicAdd(&g_prof[2], (unsigned long long)p_tf);
      atomicAdd(&g_prof[3], 1ull);
    }
#endif
  } else {
    // 16 epilogue warps.  Phase 1: TMEM lane quadrant q = warp % 4 (row m =
    // 32q + lane of the 30-wide space), channel group cg of 16 -> bias, ReLU,
    // unscale into a channel-major smem tile [64 ch][128 rows] (consecutive
    // lanes -> consecutive rows: conflict-free).  Phase 2: every epilogue
    // thread takes whole 2x2 windows (sequential argmax in q0, q1, q2, q3
    // order, strict >) and writes pooled value + code, consecutive threads ->
    // consecutive pooled positions of one channel.  Tiles alternate between
    // two smem buffers, so one named barrier per tile orders both phases.
    // (A two-group producer / consumer split of the phases measured no faster:
    // MMA operand reads, TMA and these 64 KB per tile share the SMEM bandwidth.)
    const int q = warp & 3, cg = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    const int et = threadIdx.x - 64;
    const float ws = wscale[wg];
    const uint32_t sE0 = tc::smem_u32(sP);
    int tile = 0;
    for (int b = 0; b < G; ++b) {
      const int n = n0 + b;
      if (n >= N || slot_row[n] < 0) continue;
      const float inv = 1.f / (a1scale[n] * ws);  // exact: powers of two
      float* pout = pooled + (int64_t)n * FLAT;
      uint8_t* cout = code + (int64_t)n * FLAT;
      for (int t = 0; t < FW_TILES; ++t, ++tile) {
        const int acc = tile & 1;
        const uint32_t sE = sE0 + acc * (C2 * FW_XLD * 4);
#ifdef FB_FWD_PROF
        long long p_a = clock64();
#endif
        tc::mbar_wait(&tfull[acc], (tile >> 1) & 1);
        tc::tc_fence_after();
#ifdef FB_FWD_PROF
        if (warp == 2 && lane == 0) atomicAdd(&g_prof[4], (unsigned long long)(clock64() - p_a));
#endif
        {
          const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + acc * FW_ACC + cg * 16;
          uint32_t v0[16], v1[16];
          tc::tmem_ld16(base, v0);
          tc::tmem_ld16(base + C2, v1);
          tc::tmem_ld_wait();
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&tempty[acc]);  // accumulator drained: the next tile may reuse it
#ifdef FB_FWD_NOEPI  // timing experiment only: drain TMEM, skip the pooling epilogue
          if (__uint_as_float(v0[0]) == 1.2345f) pout[0] = __uint_as_float(v1[1]);
          continue;
#endif
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j)
            v[j] = fmaxf(fmaf(__uint_as_float(v0[j]) + __uint_as_float(v1[j]), inv, bias[cg * 16 + j]), 0.f);
          // x half of the 2x2 pool in registers: rows m, m^1 are (x, x+1) of one conv row
          // (row starts are multiples of 30, even).  The even lane keeps channels 0-7 of the
          // group, the odd lane 8-15; the winner bit (x+1 strictly greater) rides in the sign
          // of the post-ReLU (>= 0) value.  Halves the epilogue's smem traffic.
          const bool odd = lane & 1;
          const uint32_t dst = sE + ((cg * 16 + (odd ? 8 : 0)) * FW_XLD + (row >> 1)) * 4;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float mine = odd ? v[8 + j] : v[j];
            const float other = __shfl_xor_sync(0xffffffffu, odd ? v[j] : v[8 + j], 1);
            const float a = odd ? other : mine, b = odd ? mine : other;  // (x, x+1)
            const bool win = b > a;
            tc::sts_f32(dst + j * FW_XLD * 4, __int_as_float(__float_as_int(win ? b : a) | ((int)win << 31)));
          }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(FW_EPI_WARPS * 32) : "memory");
        // four consecutive pooled outputs of one channel per thread: one float4 + one
        // 4-byte code store (the 28 outputs of a tile row pair start 16-byte aligned)
        for (int it = et; it < C2 * 2 * SP / 4; it += FW_EPI_WARPS * 32) {
          const int ch = it / (2 * SP / 4), pp0 = 4 * (it - ch * (2 * SP / 4));
          float best[4];
          uint32_t codes = 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int pp = pp0 + e, pr = pp >= SP, px = pp - pr * SP;
            const uint32_t e0 = sE + (ch * FW_XLD + pr * S1 + px) * 4;  // row 2pr pair px; row 2pr+1 is 15 pairs on
            const float ta = tc::lds_f32(e0), tb = tc::lds_f32(e0 + (S1 / 2) * 4);
            const float a = fabsf(ta), b = fabsf(tb);
            // first maximum in (y,x), (y,x+1), (y+1,x), (y+1,x+1) order, as the sequential scan
            const bool low = b > a;
            best[e] = low ? b : a;
            codes |= (uint32_t)(low ? 2 + (int)signbit(tb) : (int)signbit(ta)) << (8 * e);
          }
          const int idx = ch * NPOOL + FW_ROWS / 2 * t * SP + pp0;
          *reinterpret_cast<float4*>(pout + idx) = make_float4(best[0], best[1], best[2], best[3]);
          if (!shared_weights) *reinterpret_cast<uint32_t*>(cout + idx) = codes;  // (evaluation: no backward)
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc<2 * FW_ACC>(tmem);
}


// ------------------------------------------- conv2 forward on CTA pairs (cta_group::2)
// The same implicit GEMM as conv2_fwd_tc_kernel, run by a 2-CTA cluster: each pair
// step is ONE M = 256 MMA chain over two tiles (the leader's tile 2k in rows 0-127,
// the peer's tile 2k+1 in rows 128-255, each band in its own CTA's smem).  B is
// split along N: the leader holds W hi (rows 0-63 of [W hi; W lo]) and rows 0-31 of
// W hi, the peer W lo and rows 32-63 of W hi, so each SM reads half of the weight
// operand per MMA (11 KB of smem operand traffic per K step and SM instead of 14).
// Only the leader issues MMAs; both CTAs' TMA completions count on the leader's
// stage barrier; commits multicast to both CTAs; the peer's epilogue warps arrive on
// the leader's accumulator-free barrier.  Each CTA's epilogue pools its own 128 rows.
constexpr int FW2_B_TAP = 6 * 1024;                       // [64 rows W hi|lo][32 rows of W hi] x 64 B
constexpr int FW2_WBYTES = 9 * FW2_B_TAP;                 // 54 KB per CTA
constexpr int FW2_STAGES = 3;
constexpr int FW2_SMEM = 1024 + FW2_WBYTES + FW2_STAGES * FW_STAGE + FW_EPI_BYTES + 256;
constexpr uint32_t FW2_IDESC = tc::idesc_f16(256, C2);
constexpr uint32_t FW2_IDESC2 = tc::idesc_f16(256, 2 * C2);
constexpr int FW2_MAXS = 16;                              // samples per pair (G <= B <= GMAX)

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(FW_THREADS, 1) conv2_fwd_tc2_kernel(
    const __grid_constant__ CUtensorMap tm_hi, const __grid_constant__ CUtensorMap tm_lo,
    const uint8_t* __restrict__ wimg, const float* __restrict__ wscale, int shared_weights,
    const int64_t* __restrict__ slot_row, int N, int G, const float* __restrict__ theta,
    const float* __restrict__ delta, int64_t ld, int B, const float* __restrict__ a1scale,
    float* __restrict__ pooled, uint8_t* __restrict__ code) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = sm;                                        // [9][6 KB]
  uint8_t* sA = sB + FW2_WBYTES;                           // [stages][hi | lo band]
  uint8_t* sP = sA + FW2_STAGES * FW_STAGE;                 // [2][64 ch][66] x-pooled outputs
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + FW_EPI_BYTES);
  uint64_t* full = bars;                 // [stages] leader: both CTAs' bands landed (2 arrivals + bytes)
  uint64_t* empty = full + FW2_STAGES;    // [stages] per CTA: the pair's MMAs are done with the stage
  uint64_t* tfull = empty + FW2_STAGES;   // [2] per CTA: accumulator ready
  uint64_t* tempty = tfull + 2;          // [2] leader: both CTAs drained the accumulator
  uint64_t* bfull = tempty + 2;          // per CTA: this CTA's weight half landed
  uint64_t* bready = bfull + 1;          // leader: the peer's weight half landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bready + 1);
  __shared__ float bias[C2];
  __shared__ int s_list[FW2_MAXS];
  __shared__ int s_ns;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_ctarank();
  const int g = blockIdx.x >> 1;  // pair index
  const int n0 = g * G;
  {  // nothing to do: both CTAs of the pair see the same slots and leave together
    // (one slot per thread, one block-wide OR: a serial scan paid an L2 round trip per slot)
    const int b = threadIdx.x;
    if (!__syncthreads_or(b < G && n0 + b < N && slot_row[n0 + b] >= 0)) return;
  }
  const int wg = shared_weights ? 0 : n0 / B;
  const float* dc = delta ? delta + (int64_t)wg * ld : nullptr;
  if (threadIdx.x < C2) bias[threadIdx.x] = wt(theta, dc, O_B2 + threadIdx.x);
  if (threadIdx.x == 0) {
    int ns = 0;
    for (int b = 0; b < G && n0 + b < N; ++b)
      if (slot_row[n0 + b] >= 0) s_list[ns++] = n0 + b;
    s_ns = ns;
    for (int i = 0; i < FW2_STAGES; ++i) {
      tc::mbar_init(&full[i], 2);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], 2 * FW_EPI_WARPS);
    }
    tc::mbar_init(bfull, 1);
    tc::mbar_init(bready, 1);
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc2<2 * FW_ACC>(tmem_slot);
  tc::tc_fence_before();
  tc::cluster_sync();  // barriers of both CTAs initialised, TMEM allocated in both
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int T = s_ns * FW_TILES;       // tiles of the pair
  const int steps = (T + 1) >> 1;      // pair steps (the peer's last tile is a dummy when T is odd)

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&tm_hi);
      tc::tma_prefetch(&tm_lo);
      // this CTA's weight half: per tap [W hi (leader) | W lo (peer)] and rows 32*rank .. +31 of W hi
      tc::mbar_arrive_expect_tx(bfull, FW2_WBYTES);
      const uint8_t* wsrc = wimg + (int64_t)wg * WIMG_BYTES;
      for (int tap = 0; tap < 9; ++tap) {
        tc::bulk_load(sB + tap * FW2_B_TAP, wsrc + (tap * 2 + rank) * FW_B_TAP, FW_B_TAP, bfull);
        tc::bulk_load(sB + tap * FW2_B_TAP + FW_B_TAP, wsrc + tap * 2 * FW_B_TAP + rank * (FW_B_TAP / 2),
                      FW_B_TAP / 2, bfull);
      }
      const uint32_t lead_full0 = tc::mapa_shared(tc::smem_u32(full), 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int k = 0; k < steps; ++k) {
        const int ti = min(2 * k + (int)rank, T - 1);  // (a dummy tile re-reads the last band)
        const int n = s_list[ti / FW_TILES], t = ti - (ti / FW_TILES) * FW_TILES;
        tc::mbar_wait(&empty[stage], phase ^ 1);
        const uint32_t fb = lead_full0 + stage * 8;
        tc::mbar_arrive_expect_tx_cluster(fb, 2 * FW_A_TX);
        uint8_t* st_ = sA + stage * FW_STAGE;
        tc::tma_load_4d_2sm(st_, &tm_hi, 0, 0, FW_ROWS * t, n, fb);
        tc::tma_load_4d_2sm(st_ + FW_A, &tm_lo, 0, 0, FW_ROWS * t, n, fb);
        if (++stage == FW2_STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (rank == 1) {  // tell the leader this CTA's weight half is resident
      tc::mbar_wait(bfull, 0);
      if (lane == 0) tc::mbar_arrive_cluster(tc::mapa_shared(tc::smem_u32(bready), 0));
    } else {
      tc::mbar_wait(bfull, 0);
      tc::mbar_wait(bready, 0);
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t sA0 = tc::smem_u32(sA), sB0 = tc::smem_u32(sB);
      for (int k = 0; k < steps; ++k) {
        const int acc = k & 1;
        tc::mbar_wait(&tempty[acc], ((k >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem + acc * FW_ACC;
        tc::mbar_wait(&full[stage], phase);
        tc::tc_fence_after();
        if (tc::elect_one()) {
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) {
            const uint32_t ah = sA0 + stage * FW_STAGE + ((tap / 3) * S1 + tap % 3) * 64, al = ah + FW_A;
            const uint32_t b1 = sB0 + tap * FW2_B_TAP, b2 = b1 + FW_B_TAP;
            tc::mma2p_f16_ks2(d, d + C2, tc::sdesc(ah, 16, 512, 4), tc::sdesc(al, 16, 512, 4),
                              tc::sdesc(b1, 16, 512, 4), tc::sdesc(b2, 16, 512, 4), FW2_IDESC2, FW2_IDESC,
                              tap != 0);
          }
          tc::mma_commit2_mc(&empty[stage], 3);
          tc::mma_commit2_mc(&tfull[acc], 3);
        }
        __syncwarp();
        if (++stage == FW2_STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // epilogue: as conv2_fwd_tc_kernel, on this CTA's tile 2k + rank of every pair step
    const int q = warp & 3, cg = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    const int et = threadIdx.x - 64;
    const float ws = wscale[wg];
    const uint32_t sE0 = tc::smem_u32(sP);
    const uint32_t lead_tempty0 = tc::mapa_shared(tc::smem_u32(tempty), 0);
    for (int k = 0; k < steps; ++k) {
      const int acc = k & 1;
      const int ti = 2 * k + (int)rank;
      const bool real = ti < T;
      const int n = real ? s_list[ti / FW_TILES] : 0, t = ti - (ti / FW_TILES) * FW_TILES;
      const uint32_t sE = sE0 + acc * (C2 * FW_XLD * 4);
      tc::mbar_wait(&tfull[acc], (k >> 1) & 1);
      tc::tc_fence_after();
      uint32_t v0[16], v1[16];
      if (real) {
        const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + acc * FW_ACC + cg * 16;
        tc::tmem_ld16(base, v0);
        tc::tmem_ld16(base + C2, v1);
        tc::tmem_ld_wait();
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster(lead_tempty0 + acc * 8);  // accumulator drained (pair-wide)
      if (!real) continue;  // (uniform across the CTA: no named barrier below for a dummy tile)
      const float inv = 1.f / (a1scale[n] * ws);  // exact: powers of two
      {
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          v[j] = fmaxf(fmaf(__uint_as_float(v0[j]) + __uint_as_float(v1[j]), inv, bias[cg * 16 + j]), 0.f);
        const bool odd = lane & 1;
        const uint32_t dst = sE + ((cg * 16 + (odd ? 8 : 0)) * FW_XLD + (row >> 1)) * 4;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float mine = odd ? v[8 + j] : v[j];
          const float other = __shfl_xor_sync(0xffffffffu, odd ? v[j] : v[8 + j], 1);
          const float a = odd ? other : mine, b = odd ? mine : other;
          const bool win = b > a;
          tc::sts_f32(dst + j * FW_XLD * 4, __int_as_float(__float_as_int(win ? b : a) | ((int)win << 31)));
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(FW_EPI_WARPS * 32) : "memory");
      float* pout = pooled + (int64_t)n * FLAT;
      uint8_t* cout = code + (int64_t)n * FLAT;
      for (int it = et; it < C2 * 2 * SP; it += FW_EPI_WARPS * 32) {
        const int ch = it / (2 * SP), pp = it - ch * (2 * SP), pr = pp >= SP, px = pp - pr * SP;
        const uint32_t e0 = sE + (ch * FW_XLD + pr * S1 + px) * 4;
        const float ta = tc::lds_f32(e0), tb = tc::lds_f32(e0 + (S1 / 2) * 4);
        const float a = fabsf(ta), b = fabsf(tb);
        const bool low = b > a;
        const float best = low ? b : a;
        const int arg = low ? 2 + (int)signbit(tb) : (int)signbit(ta);
        const int idx = ch * NPOOL + FW_ROWS / 2 * t * SP + pp;
        pout[idx] = best;
        cout[idx] = (uint8_t)arg;
      }
    }
  }
  tc::tc_fence_before();
  tc::cluster_sync();  // both CTAs done with the pair's TMEM and barriers
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc2<2 * FW_ACC>(tmem);
}

// ------------------------------------------------------- fc1 on tcgen05
// Both fc1 contractions of the factored form run at theta_t, i.e. as plain
// GEMMs over all slots of the step (kind::f16, 3-term split as above):
//   forward   part[sp][n][h] = sum_{k in split sp} P[n][k] W[k][h]   (M = slots, N = 128, K = 12544)
//   backward  dp[n][k]       = sum_h dz3[n][h] W[k][h]              (M = slots, N = 12544, K = 128)
// One persistent kernel serves both: a work unit is one 128-row M tile x 128
// output columns over a run of 64-wide K stages; each stage is four TMA
// boxes (A hi / lo, B hi / lo: 128 rows x 128 B, SWIZZLE_128B) and 12 UMMAs
// 128x128x16.  The TMEM accumulators (hi*hi and the two cross terms
// separately) are drained every FT_WIN stages by the epilogue warps into
// fp32 registers (round-to-nearest), double-buffered so the drain overlaps
// the next window's MMAs -- the tensor core's own long accumulation chains
// are not accurate enough for the 12544-long forward sum.  The operands are
// scaled per row (slot) and per matrix (theta) by powers of two; the
// epilogue unscales exactly.
constexpr int FT_KS = 64;                              // K per stage (64 fp16 = one 128 B swizzle row)
constexpr int FT_PART = 128 * 128;                     // 16 KB: 128 rows x 64 fp16
constexpr int FT_STAGE = 4 * FT_PART;                  // A hi, A lo, B hi, B lo
constexpr int FT_STAGES = 3;
constexpr int FT_WIN = 2;                              // stages per accumulation window
constexpr int FT_FSPLIT = 14;                          // forward K split: 12544 = 14 x 896
constexpr int FT_FSTAGES = FLAT / FT_FSPLIT / FT_KS;   // 14 stages per forward unit
constexpr int FT_BSTAGES = HID / FT_KS;                // 2 stages per backward unit
constexpr int FT_SMEM = 1024 + FT_STAGES * FT_STAGE + 256;
constexpr uint32_t FT_IDESC = tc::idesc_f16(128, 128);
static_assert(FLAT % (FT_FSPLIT * FT_KS) == 0, "fc1 forward split");
static_assert(FT_FSTAGES % FT_WIN == 0 && FT_BSTAGES % FT_WIN == 0, "fc1 windows");
static_assert(FLAT % 128 == 0, "fc1 backward N tiles");

// max |W_fc1| (float bits of a non-negative value compare as unsigned)
__global__ void __launch_bounds__(256) fc1_theta_max_kernel(const float* __restrict__ theta,
                                                            unsigned* __restrict__ tmax) {
  float m = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)FLAT * HID;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(theta[O_F1 + i]));
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomicMax(tmax, __float_as_uint(m));
}

// fp16 hi / lo images of W_fc1 * tscale: thT[h][k] (forward B operand, K = k)
// and th[k][h] (backward B operand, K = h); one CTA per 64 rows of k
__global__ void __launch_bounds__(256) fc1_theta_img_kernel(const float* __restrict__ theta,
                                                            const unsigned* __restrict__ tmax,
                                                            __half* __restrict__ thTh, __half* __restrict__ thTl,
                                                            __half* __restrict__ thh, __half* __restrict__ thl,
                                                            float* __restrict__ tscale) {
  __shared__ float tile[64][HID + 1];
  const float m = __uint_as_float(*tmax);
  const float sc = m > 0.f ? exp2f(14.f - ceilf(log2f(m))) : 1.f;
  if (blockIdx.x == 0 && threadIdx.x == 0) *tscale = sc;
  const int k0 = blockIdx.x * 64;
  for (int i = threadIdx.x; i < 64 * HID; i += blockDim.x) {
    const int r = i / HID, h = i - r * HID;
    const int64_t o = (int64_t)(k0 + r) * HID + h;
    const float v = theta[O_F1 + o] * sc;
    tile[r][h] = v;
    __half hh, ll;
    split_f16(v, hh, ll);
    thh[o] = hh;
    thl[o] = ll;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 64 * HID; i += blockDim.x) {
    const int h = i / 64, r = i - h * 64;
    __half hh, ll;
    split_f16(tile[r][h], hh, ll);
    thTh[(int64_t)h * FLAT + k0 + r] = hh;
    thTl[(int64_t)h * FLAT + k0 + r] = ll;
  }
}

// pooled activations -> per-slot scaled fp16 hi / lo (forward A operand)
__global__ void __launch_bounds__(256) pooled_split_kernel(const float* __restrict__ pooled,
                                                           const int64_t* __restrict__ slot_row,
                                                           __half* __restrict__ ph, __half* __restrict__ pl,
                                                           float* __restrict__ pscale) {
  __shared__ float red[32];
  const int n = blockIdx.x;
  if (slot_row[n] < 0) {  // inactive slot: zero operand rows (the factored fc1 history reads every slot)
    uint2* dh = reinterpret_cast<uint2*>(ph + (int64_t)n * FLAT);
    uint2* dl = reinterpret_cast<uint2*>(pl + (int64_t)n * FLAT);
    for (int i = threadIdx.x; i < FLAT / 4; i += blockDim.x) dh[i] = dl[i] = make_uint2(0u, 0u);
    if (threadIdx.x == 0) pscale[n] = 1.f;
    return;
  }
  // the row is held in registers between the max pass and the split (one HBM read, all
  // loads of a thread in flight together); 256 threads x PS_Q float4 cover the 12544 values
  constexpr int PS_Q = (FLAT / 4 + 255) / 256;
  const float4* src = reinterpret_cast<const float4*>(pooled + (int64_t)n * FLAT);
  float4 v[PS_Q];
  float m = 0.f;
#pragma unroll
  for (int u = 0; u < PS_Q; ++u) {
    const int i = threadIdx.x + u * 256;
    v[u] = i < FLAT / 4 ? __ldg(src + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
  }
  const float sc = block_scale(m, red);
  if (threadIdx.x == 0) pscale[n] = sc;
  uint2* dh = reinterpret_cast<uint2*>(ph + (int64_t)n * FLAT);
  uint2* dl = reinterpret_cast<uint2*>(pl + (int64_t)n * FLAT);
#pragma unroll
  for (int u = 0; u < PS_Q; ++u) {
    const int i = threadIdx.x + u * 256;
    if (i < FLAT / 4) {
      uint32_t a, b, c, d;
      split_f16x2(v[u].x * sc, v[u].y * sc, a, c);
      split_f16x2(v[u].z * sc, v[u].w * sc, b, d);
      dh[i] = make_uint2(a, b);
      dl[i] = make_uint2(c, d);
    }
  }
}

struct FtArgs {
  int mode;               // 0 = forward (part), 1 = backward (dp)
  int N;                  // slots (A rows)
  int mtiles, units;
  const float* rscale;    // per-slot operand scale (pooled / dz3)
  const float* tscale;    // W_fc1 scale
  float* out;
};

__global__ void __launch_bounds__(TC_THREADS, 1) fc1_tc_kernel(const __grid_constant__ CUtensorMap ta_h,
                                                               const __grid_constant__ CUtensorMap ta_l,
                                                               const __grid_constant__ CUtensorMap tb_h,
                                                               const __grid_constant__ CUtensorMap tb_l, FtArgs fa) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + FT_STAGES * FT_STAGE);
  uint64_t* full = bars;
  uint64_t* empty = bars + FT_STAGES;
  uint64_t* tfull = empty + FT_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nst = fa.mode == 0 ? FT_FSTAGES : FT_BSTAGES;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < FT_STAGES; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], 4);
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // unit -> (A row, B row, first K, output)
  auto unit_geom = [&](int u, int& arow, int& brow, int& kb, int& sp_or_nt) {
    if (fa.mode == 0) {
      const int mt = u / FT_FSPLIT;
      sp_or_nt = u - mt * FT_FSPLIT;
      arow = mt * 128;
      brow = 0;
      kb = sp_or_nt * FT_FSTAGES * FT_KS;
    } else {
      const int nt = u / fa.mtiles;
      sp_or_nt = nt;
      arow = (u - nt * fa.mtiles) * 128;
      brow = nt * 128;
      kb = 0;
    }
  };

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&ta_h);
      tc::tma_prefetch(&ta_l);
      tc::tma_prefetch(&tb_h);
      tc::tma_prefetch(&tb_l);
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < fa.units; u += gridDim.x) {
        int arow, brow, kb, x;
        unit_geom(u, arow, brow, kb, x);
        for (int st_ = 0; st_ < nst; ++st_) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          tc::mbar_arrive_expect_tx(&full[stage], FT_STAGE);
          uint8_t* d = sm + stage * FT_STAGE;
          const int k = kb + st_ * FT_KS;
          tc::tma_load_2d(d, &ta_h, k, arow, &full[stage]);
          tc::tma_load_2d(d + FT_PART, &ta_l, k, arow, &full[stage]);
          tc::tma_load_2d(d + 2 * FT_PART, &tb_h, k, brow, &full[stage]);
          tc::tma_load_2d(d + 3 * FT_PART, &tb_l, k, brow, &full[stage]);
          if (++stage == FT_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    int stage = 0, win = 0;
    uint32_t phase = 0;
    const uint32_t s0 = tc::smem_u32(sm);
    for (int u = blockIdx.x; u < fa.units; u += gridDim.x) {
      for (int st_ = 0; st_ < nst; ++st_) {
        const int buf = win & 1;
        if (st_ % FT_WIN == 0) {
          tc::mbar_wait(&tempty[buf], ((win >> 1) & 1) ^ 1);
          tc::tc_fence_after();
        }
        tc::mbar_wait(&full[stage], phase);
        tc::tc_fence_after();
        if (tc::elect_one()) {
          const uint32_t ah = s0 + stage * FT_STAGE, al = ah + FT_PART, bh = ah + 2 * FT_PART, bl = ah + 3 * FT_PART;
          const uint32_t dmain = tmem + buf * 256, dcross = dmain + 128;
          static_assert(FT_KS == 64, "fc1 stage = 4 K steps");
          const uint32_t acc = st_ % FT_WIN != 0 ? 1u : 0u;  // a window's first stage starts fresh accumulators
          tc::mma3_f16_ks<4, 2, 2>(dmain, dcross, tc::sdesc(ah, 16, 1024, 2), tc::sdesc(al, 16, 1024, 2),
                                   tc::sdesc(bh, 16, 1024, 2), tc::sdesc(bl, 16, 1024, 2), FT_IDESC, acc, acc);
          tc::mma_commit(&empty[stage]);
          if (st_ % FT_WIN == FT_WIN - 1) tc::mma_commit(&tfull[buf]);
        }
        __syncwarp();
        if (st_ % FT_WIN == FT_WIN - 1) ++win;
        if (++stage == FT_STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    const int ew = warp & 3;
    const int row = ew * 32 + lane;
    const float ts = *fa.tscale;
    int win = 0;
    for (int u = blockIdx.x; u < fa.units; u += gridDim.x) {
      int arow, brow, kb, x;
      unit_geom(u, arow, brow, kb, x);
      float sum[128];
#pragma unroll
      for (int i = 0; i < 128; ++i) sum[i] = 0.f;
      for (int w = 0; w < nst / FT_WIN; ++w, ++win) {
        const int buf = win & 1;
        tc::mbar_wait(&tfull[buf], (win >> 1) & 1);
        tc::tc_fence_after();
        const uint32_t base = tmem + ((uint32_t)(ew * 32) << 16) + buf * 256;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t v0[32], v1[32];
          tc::tmem_ld32(base + q * 32, v0);
          tc::tmem_ld32(base + 128 + q * 32, v1);
          tc::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) sum[q * 32 + i] += __uint_as_float(v0[i]) + __uint_as_float(v1[i]);
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&tempty[buf]);
      }
      const int n = arow + row;
      if (n < fa.N) {
        const float inv = 1.f / (fa.rscale[n] * ts);
        float* o = fa.mode == 0 ? fa.out + ((int64_t)x * fa.N + n) * HID
                                : fa.out + (int64_t)n * FLAT + (int64_t)x * 128;
        // 256-bit stores: the row-per-lane pattern writes one FULL 32-byte sector per lane and
        // instruction (16-byte stores left every L2 write sector half-filled: 2x the write
        // sectors, ncu r02cp)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          uint32_t v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = __float_as_uint(sum[8 * i + e] * inv);
          stg256(o + 8 * i, v);
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc<512>(tmem);
}

int tensor_map_2d_f16(CUtensorMap* map, const __half* base, int64_t inner, int64_t rows, int box_inner, int box_rows) {
  auto fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return FB_ERR_CUDA;
  }
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)inner * 2};
  const cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (2-D fp16) failed (%d)", (int)r);
    return FB_ERR_CUDA;
  }
  return FB_OK;
}

// dp -= sum_j a[b][j] p_j (history part of the factored backward); grid (C, KSPLIT),
// thread = 4 k.  The client's active history rows are compacted first so the row loop
// has no branch and issues four independent float4 loads per trip.
#ifndef DPH_U
#define DPH_U 4  // history rows loaded per trip of fc1_dp_hist_kernel
#endif
template <int GM>
__global__ void __launch_bounds__(KCHUNK / 4) fc1_dp_hist_kernel(int B, const int32_t* __restrict__ client_nb, Hist hs,
                                                                 float* __restrict__ dp) {
  __shared__ float ac[FC_RMAX * GMAX];  // [compact row q][b]
  __shared__ uint32_t roff[FC_RMAX];
  __shared__ int jsrc[FC_RMAX];
  __shared__ int s_cnt[2];
  const int c = blockIdx.x, k0 = blockIdx.y * KCHUNK, t = threadIdx.x;
  const int nb = client_nb[c];
  const int J = hs.s * B;
  if (nb == 0 || J == 0) return;
  const int n0 = c * B;
  // compact the active history rows in parallel (J <= 64: warps 0 and 1, ballot + popc),
  // keeping row order; a serial scan here cost one dependent L2 round trip per row
  static_assert(FC_RMAX <= 64 && KCHUNK / 4 >= 64, "dp_hist compaction: two warps");
  bool act = false;
  int sp = 0, bp = 0;
  if (t < 64) {
    sp = t / B;
    bp = t - sp * B;
    act = t < J && bp < hs.nbh[sp * hs.cstride + c];
  }
  const unsigned bal = t < 64 ? __ballot_sync(0xffffffffu, act) : 0u;
  if (t < 64 && (t & 31) == 0) s_cnt[t >> 5] = __popc(bal);
  __syncthreads();
  if (act) {
    const int q = (t >= 32 ? s_cnt[0] : 0) + __popc(bal & ((1u << (t & 31)) - 1u));
    jsrc[q] = t;
    roff[q] = (uint32_t)(sp * hs.pstride + (int64_t)(n0 + bp) * FLAT + k0);  // host checks S*N*FLAT < 2^31
  }
  __syncthreads();
  const int nj = s_cnt[0] + s_cnt[1];
  for (int i = t; i < nj * GM; i += blockDim.x) {
    const int q = i / GM, b = i - q * GM;
    ac[i] = b < nb ? hs.acoef[((int64_t)c * GMAX + b) * FC_RMAX + jsrc[q]] : 0.f;
  }
  __syncthreads();
  float4 acc[GM];
#pragma unroll
  for (int b = 0; b < GM; ++b)
    acc[b] = b < nb ? reinterpret_cast<const float4*>(dp + (int64_t)(n0 + b) * FLAT + k0)[t]
                    : make_float4(0.f, 0.f, 0.f, 0.f);
  const float4* ph = reinterpret_cast<const float4*>(hs.phist);
  int q = 0;
#pragma unroll 1
  for (; q + DPH_U <= nj; q += DPH_U) {
    float4 p[DPH_U];
#pragma unroll
    for (int u = 0; u < DPH_U; ++u) p[u] = __ldg(ph + (roff[q + u] >> 2) + t);
#pragma unroll
    for (int u = 0; u < DPH_U; ++u)
#pragma unroll
      for (int b = 0; b < GM; ++b) {
        const float a = ac[(q + u) * GM + b];
        acc[b].x = fmaf(-a, p[u].x, acc[b].x);
        acc[b].y = fmaf(-a, p[u].y, acc[b].y);
        acc[b].z = fmaf(-a, p[u].z, acc[b].z);
        acc[b].w = fmaf(-a, p[u].w, acc[b].w);
      }
  }
#pragma unroll 1
  for (; q < nj; ++q) {
    const float4 p = __ldg(ph + (roff[q] >> 2) + t);
#pragma unroll
    for (int b = 0; b < GM; ++b) {
      const float a = ac[q * GM + b];
      acc[b].x = fmaf(-a, p.x, acc[b].x);
      acc[b].y = fmaf(-a, p.y, acc[b].y);
      acc[b].z = fmaf(-a, p.z, acc[b].z);
      acc[b].w = fmaf(-a, p.w, acc[b].w);
    }
  }
#pragma unroll
  for (int b = 0; b < GM; ++b)
    if (b < nb) reinterpret_cast<float4*>(dp + (int64_t)(n0 + b) * FLAT + k0)[t] = acc[b];
}

// ----------------------------------------- fc1 materialize (tcgen05)
// End of a factored-fc1 run: delta_fc1[c][k][h] = sum_j coef_j dz3_j[h] p_j[k]
// over the client's <= 64 history rows j = (step s, slot b).  A GEMM per
// client with M = k (98 tiles of 128), N = h (128), K = j (64 = 4 x 16):
// A = P^T from the fp16 hi / lo pooled history the tcgen05 fc1 forward
// already wrote (per-row power-of-two scale pscale_j), MN-major: one 3-D TMA
// box {64 k, B slots, S steps} per 64-wide M block lands the client's rows
// j = s*B + b as consecutive 128-byte K rows; B = U' = coef_j dz3_j /
// pscale_j * beta (beta: per-client power of two), built once per CTA and
// split hi / lo, stacked along N ([U hi | U lo], N = 256) so per K step one
// N = 256 and one N = 128 MMA form the three split products.  TMEM tiles
// (main | cross, 256 columns) are double-buffered; 8 epilogue warps sum,
// unscale and write the client's fp32 fc1 delta (6.4 MB, the HBM floor).
constexpr int FMT_TILE = 128;
constexpr int FMT_TILES = FLAT / FMT_TILE;        // 98
constexpr int FMT_SPLIT = 2;                      // CTAs per client: 49 tiles each (U' built twice per client)
constexpr int FMT_BLK = FC_RMAX * 128;            // 8 KB: 64 j rows x 64 fp16
constexpr int FMT_STAGE = 4 * FMT_BLK;            // A hi (2 M blocks) | A lo (2 M blocks)
constexpr int FMT_STAGES = 3;
constexpr int FMT_BOP = 4 * FMT_BLK;              // U hi (2 N blocks) | U lo (2 N blocks)
constexpr int FMT_EPI_WARPS = 8;
constexpr int FMT_THREADS = (2 + FMT_EPI_WARPS) * 32;
constexpr int FMT_SMEM = 1024 + FMT_BOP + FMT_STAGES * FMT_STAGE + 256 + FMT_EPI_WARPS * 32 * 33 * 4;
constexpr uint32_t FMT_IDESC2 = tc::idesc_f16_mn(128, 2 * HID);
constexpr uint32_t FMT_IDESC = tc::idesc_f16_mn(128, HID);
static_assert(FLAT % FMT_TILE == 0 && FMT_TILES % FMT_SPLIT == 0 && FMT_TILES % 7 == 0, "fc1 materialize tiles");

// 3-D fp16 map of the pooled history [S][N][FLAT]: box {64 k, B slots, S steps}
int hist_tensor_map(CUtensorMap* map, const __half* base, int N, int S, int B) {
  auto fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return FB_ERR_CUDA;
  }
  const cuuint64_t dims[3] = {(cuuint64_t)FLAT, (cuuint64_t)N, (cuuint64_t)S};
  const cuuint64_t strides[2] = {(cuuint64_t)FLAT * 2, (cuuint64_t)N * FLAT * 2};
  const cuuint32_t box[3] = {64, (cuuint32_t)B, (cuuint32_t)S};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<__half*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (3-D history) failed (%d)", (int)r);
    return FB_ERR_CUDA;
  }
  return FB_OK;
}

__global__ void __launch_bounds__(FMT_THREADS, 1) fc1_mat_tc_kernel(
    const __grid_constant__ CUtensorMap tm_hi, const __grid_constant__ CUtensorMap tm_lo, Hist hs,
    const float* __restrict__ pscale_hist, int N, int S, int B, float lr, float mu, float* __restrict__ delta,
    int64_t ld, double* __restrict__ sumsq_part, int store) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = sm;                                  // [U hi blk0 | U hi blk1 | U lo blk0 | U lo blk1]
  uint8_t* sA = sm + FMT_BOP;                        // [stage][hi blk0 | hi blk1 | lo blk0 | lo blk1]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + FMT_STAGES * FMT_STAGE);
  uint64_t* full = bars;
  uint64_t* empty = full + FMT_STAGES;
  uint64_t* tfull = empty + FMT_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ float red[32];
  __shared__ double red_sq[FMT_EPI_WARPS];
  __shared__ int s_sc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = threadIdx.x;
  const int nt = FMT_TILES / gridDim.y;  // tiles per CTA (gridDim.y divides 98)
  const int c = blockIdx.x, t0 = blockIdx.y * nt;
  const int J = S * B;
  if (t == 0) {
    int Sc = 0;
    while (Sc < S && hs.nbh[Sc * hs.cstride + c] > 0) ++Sc;
    s_sc = Sc;
  }
  __syncthreads();
  const int Sc = s_sc;
  if (Sc == 0) {  // the client never trained (no rows): its fc1 delta block is zero (zero_delta skipped it)
    if (!store) {
      if (sumsq_part && t == 0) sumsq_part[(int64_t)c * gridDim.y + blockIdx.y] = 0.0;
      return;
    }
    float4* z = reinterpret_cast<float4*>(delta + (int64_t)c * ld + O_F1 + (int64_t)t0 * FMT_TILE * HID);
    for (int i = t; i < nt * FMT_TILE * HID / 4; i += FMT_THREADS) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  // U' rows j = s*B + b (zero when inactive); per-client power-of-two beta puts max |U'| at ~2^14.
  // The thread's values stay in registers between the max pass and the split (all loads of
  // the thread in flight together instead of one L2 round trip per element and pass).
  constexpr int UQ = (FC_RMAX * HID + FMT_THREADS - 1) / FMT_THREADS;
  float uv[UQ];
  float m = 0.f;
#pragma unroll
  for (int u = 0; u < UQ; ++u) {
    const int i = t + u * FMT_THREADS;
    const int j = i / HID, h = i - j * HID, sp = j / B, bp = j - sp * B;
    float v = 0.f;
    if (i < FC_RMAX * HID && j < J && sp < Sc && bp < hs.nbh[sp * hs.cstride + c]) {
      const int64_t slot = (int64_t)c * B + bp;
      v = hist_coef(lr, mu, Sc, sp) * hs.dz3h[sp * hs.dstride + slot * HID + h] / pscale_hist[(int64_t)sp * N + slot];
    }
    uv[u] = v;
    m = fmaxf(m, fabsf(v));
  }
  const float beta = block_scale(m, red);
#pragma unroll
  for (int u = 0; u < UQ; ++u) {
    const int i = t + u * FMT_THREADS;
    if (i >= FC_RMAX * HID) break;
    const int j = i / HID, h = i - j * HID;
    __half hi, lo;
    split_f16(uv[u] * beta, hi, lo);
    const uint32_t off = (h >> 6) * FMT_BLK + sw128_off16(j, h & 63);
    *reinterpret_cast<__half*>(sB + off) = hi;
    *reinterpret_cast<__half*>(sB + 2 * FMT_BLK + off) = lo;
  }
  // A rows J..63 of every stage / block stay zero (the TMA box fills rows 0..J-1 only)
  for (int st = 0; st < FMT_STAGES; ++st)
    for (int i = t; i < 4 * (FC_RMAX - J) * 32; i += FMT_THREADS) {
      const int blk = i / ((FC_RMAX - J) * 32), r = i - blk * (FC_RMAX - J) * 32;
      reinterpret_cast<uint32_t*>(sA + st * FMT_STAGE + blk * FMT_BLK + J * 128)[r] = 0u;
    }
  if (t == 0) {
    for (int i = 0; i < FMT_STAGES; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], FMT_EPI_WARPS);
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(tmem_slot);
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&tm_hi);
      tc::tma_prefetch(&tm_lo);
      int stage = 0;
      uint32_t phase = 0;
      for (int ti = 0; ti < nt; ++ti) {
        const int k0 = (t0 + ti) * FMT_TILE;
        tc::mbar_wait(&empty[stage], phase ^ 1);
        tc::mbar_arrive_expect_tx(&full[stage], 4 * J * 128);
        uint8_t* st_ = sA + stage * FMT_STAGE;
        tc::tma_load_3d(st_, &tm_hi, k0, c * B, 0, &full[stage]);
        tc::tma_load_3d(st_ + FMT_BLK, &tm_hi, k0 + 64, c * B, 0, &full[stage]);
        tc::tma_load_3d(st_ + 2 * FMT_BLK, &tm_lo, k0, c * B, 0, &full[stage]);
        tc::tma_load_3d(st_ + 3 * FMT_BLK, &tm_lo, k0 + 64, c * B, 0, &full[stage]);
        if (++stage == FMT_STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t sA0 = tc::smem_u32(sA), sB0 = tc::smem_u32(sB);
    for (int ti = 0; ti < nt; ++ti) {
      const int acc = ti & 1;
      tc::mbar_wait(&tempty[acc], ((ti >> 1) & 1) ^ 1);
      tc::tc_fence_after();
      tc::mbar_wait(&full[stage], phase);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint32_t d = tmem + acc * 256;
        const uint32_t ah = sA0 + stage * FMT_STAGE, al = ah + 2 * FMT_BLK;
#pragma unroll
        for (int ks = 0; ks < FC_RMAX / 16; ++ks) {  // 16 history rows = two 8-row K atoms per step
          const uint64_t adh = tc::sdesc(ah + ks * 2048, FMT_BLK, 1024, 2);
          const uint64_t adl = tc::sdesc(al + ks * 2048, FMT_BLK, 1024, 2);
          const uint64_t bd = tc::sdesc(sB0 + ks * 2048, FMT_BLK, 1024, 2);
          tc::mma2_f16(d, d + HID, adh, adl, bd, FMT_IDESC2, FMT_IDESC, ks != 0);
        }
        tc::mma_commit(&empty[stage]);
        tc::mma_commit(&tfull[acc]);
      }
      __syncwarp();
      if (++stage == FMT_STAGES) { stage = 0; phase ^= 1; }
    }
  } else {
    const int q = warp & 3, hh = (warp - 2) >> 2;  // TMEM lane quadrant, h half
    const float inv = 1.f / beta;                   // exact: power of two
    float* dc = delta + (int64_t)c * ld + O_F1;
    // per-warp 32 x 33 transpose tile: lane = k row in TMEM; the stores go out as
    // 4 rows x 128 contiguous bytes per instruction instead of 32 rows x 16 B
    const uint32_t tw = tc::smem_u32(sA + FMT_STAGES * FMT_STAGE + 256) + (warp - 2) * 32 * 33 * 4;
    double sq = 0.0;  // sum of squares of this thread's stored values (fixed order)
    for (int ti = 0; ti < nt; ++ti) {
      const int acc = ti & 1;
      tc::mbar_wait(&tfull[acc], (ti >> 1) & 1);
      tc::tc_fence_after();
      const int kbase = (t0 + ti) * FMT_TILE + q * 32;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + acc * 256 + hh * 64 + half * 32;
        uint32_t v0[32], v1[32];
        tc::tmem_ld32(base, v0);
        tc::tmem_ld32(base + HID, v1);
        tc::tmem_ld_wait();
        if (half == 1) {
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&tempty[acc]);
        }
        if (!store) {  // squares only (the factored aggregate never materialises the block):
          // four independent fp32 chains of 8 per half, then one fp64 add
          float q4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float z = (__uint_as_float(v0[j]) + __uint_as_float(v1[j])) * inv;
            q4[j & 3] = fmaf(z, z, q4[j & 3]);
          }
          sq += (double)((q4[0] + q4[1]) + (q4[2] + q4[3]));
          continue;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float z = (__uint_as_float(v0[j]) + __uint_as_float(v1[j])) * inv;
          sq = fma((double)z, (double)z, sq);
          tc::sts_f32(tw + (lane * 33 + j) * 4, z);
        }
        __syncwarp();
        const int r = lane >> 3, c4 = (lane & 7) * 4;
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
          const int row = rr * 4 + r;
          float4 o;
          o.x = tc::lds_f32(tw + (row * 33 + c4) * 4);
          o.y = tc::lds_f32(tw + (row * 33 + c4 + 1) * 4);
          o.z = tc::lds_f32(tw + (row * 33 + c4 + 2) * 4);
          o.w = tc::lds_f32(tw + (row * 33 + c4 + 3) * 4);
          *reinterpret_cast<float4*>(dc + (int64_t)(kbase + row) * HID + hh * 64 + half * 32 + c4) = o;
        }
        __syncwarp();
      }
    }
    if (sumsq_part) {  // per-CTA partial: warp tree, then the 8 warps in order
      sq = warp_sum(sq);
      if (lane == 0) red_sq[warp - 2] = sq;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (sumsq_part && threadIdx.x == 0) {
    double tot = 0.0;
    for (int i = 0; i < FMT_EPI_WARPS; ++i) tot += red_sq[i];
    sumsq_part[(int64_t)c * gridDim.y + blockIdx.y] = tot;
  }
  if (warp == 1) tc::tmem_dealloc<512>(tmem);
}

// ------------------------------------------- factored fc1 aggregate (tcgen05)
// K3 for the fc1 weight block without materialising any client's delta:
//   agg[k][h] = sum_c coef_c delta_c[k][h] = sum_c sum_j p_cj[k] U'_cj[h],
//   U'_cj = coef_c * hist_coef_j * dz3_cj / pscale_cj,
// one GEMM with M = k (98 tiles of 128), N = h (128) and K = every history row of
// the cohort.  U' is built once per client (fp16 hi / lo with ONE cohort-wide
// power-of-two scale so clients accumulate in the same TMEM tile) and streamed by
// TMA with the pooled-history tiles; a CTA owns one k tile and a chunk of clients,
// drains its accumulator every FAG_DRAIN clients (32-step chains) into fp32
// registers and writes a per-chunk partial; fc1_agg_reduce_kernel sums the chunks in
// fixed order.  Reads 2.5 GB of history instead of writing + re-reading the 6.4 GB of
// per-client fc1 deltas.  (Clip norms come from fc1_mat_tc_kernel in squares-only mode.)
#ifndef FAG_NCHUNKS
#define FAG_NCHUNKS 6  // 588 CTAs: ~4 full waves on 148 SMs (measured 0.47 vs 0.53 ms at 8)
#endif
constexpr int FAG_CHUNKS = FAG_NCHUNKS;                // client chunks (grid.y)
constexpr int FAG_DRAIN = 8;                           // clients per TMEM accumulation chain
constexpr int FAG_UBYTES = 4 * FMT_BLK;                // U' hi blk0 | blk1 | lo blk0 | blk1 (32 KB)
constexpr int FAG_STAGE = FMT_STAGE + FAG_UBYTES;      // P tile (32 KB) + U' (32 KB)
constexpr int FAG_STAGES = 3;
constexpr int FAG_SMEM = 1024 + FAG_STAGES * FAG_STAGE + 256;

// cohort max |U'| (float bits of a non-negative value compare as unsigned)
__global__ void __launch_bounds__(256) fc1_umax_kernel(Hist hs, const float* __restrict__ pscale_hist,
                                                       const float* __restrict__ coef, int N, int S, int B,
                                                       float lr, float mu, unsigned* __restrict__ umax) {
  const int c = blockIdx.x;
  int Sc = 0;
  while (Sc < S && hs.nbh[Sc * hs.cstride + c] > 0) ++Sc;
  float m = 0.f;
  const float k = coef[c];
  for (int i = threadIdx.x; i < S * B * HID; i += blockDim.x) {
    const int j = i / HID, h = i - j * HID, sp = j / B, bp = j - sp * B;
    if (sp < Sc && bp < hs.nbh[sp * hs.cstride + c]) {
      const int64_t slot = (int64_t)c * B + bp;
      m = fmaxf(m, fabsf(k * hist_coef(lr, mu, Sc, sp) * hs.dz3h[sp * hs.dstride + slot * HID + h] /
                         pscale_hist[(int64_t)sp * N + slot]));
    }
  }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomicMax(umax, __float_as_uint(m));
}

// U' of client c as fp16 hi / lo, [c][hi|lo][64 rows j][128 h] (rows past the client's
// history and inactive slots zero), scaled by the cohort-wide power of two
__global__ void __launch_bounds__(256) fc1_ubuild_kernel(Hist hs, const float* __restrict__ pscale_hist,
                                                         const float* __restrict__ coef, int N, int S, int B,
                                                         float lr, float mu, const unsigned* __restrict__ umax,
                                                         __half* __restrict__ u) {
  const int c = blockIdx.x;
  int Sc = 0;
  while (Sc < S && hs.nbh[Sc * hs.cstride + c] > 0) ++Sc;
  const float m = __uint_as_float(*umax);
  const float beta = m > 0.f ? exp2f(14.f - ceilf(log2f(m))) : 1.f;
  const float k = coef[c] * beta;
  __half* uh = u + (int64_t)c * 2 * FC_RMAX * HID;
  __half* ul = uh + FC_RMAX * HID;
  for (int i = threadIdx.x; i < FC_RMAX * HID / 2; i += blockDim.x) {
    const int j = (2 * i) / HID, h = 2 * i - j * HID, sp = j / B, bp = j - sp * B;
    float v0 = 0.f, v1 = 0.f;
    if (j < S * B && sp < Sc && bp < hs.nbh[sp * hs.cstride + c]) {
      const int64_t slot = (int64_t)c * B + bp;
      const float f = k * hist_coef(lr, mu, Sc, sp) / pscale_hist[(int64_t)sp * N + slot];
      v0 = f * hs.dz3h[sp * hs.dstride + slot * HID + h];
      v1 = f * hs.dz3h[sp * hs.dstride + slot * HID + h + 1];
    }
    uint32_t hw, lw;
    split_f16x2(v0, v1, hw, lw);
    reinterpret_cast<uint32_t*>(uh)[i] = hw;
    reinterpret_cast<uint32_t*>(ul)[i] = lw;
  }
}

__global__ void __launch_bounds__(FMT_THREADS, 1) fc1_agg_tc_kernel(
    const __grid_constant__ CUtensorMap tm_hi, const __grid_constant__ CUtensorMap tm_lo,
    const __grid_constant__ CUtensorMap tm_u, int C, int S, int B, int chunk, const unsigned* __restrict__ umax,
    float* __restrict__ part) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;  // [stage][P hi blk0 | blk1 | P lo blk0 | blk1 | U hi blk0 | blk1 | U lo blk0 | blk1]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + FAG_STAGES * FAG_STAGE);
  uint64_t* full = bars;
  uint64_t* empty = full + FAG_STAGES;
  uint64_t* tfull = empty + FAG_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = threadIdx.x;
  const int kt = blockIdx.x, c0 = blockIdx.y * chunk, c1 = min(C, c0 + chunk), nc = c1 - c0;
  const int J = S * B;
  float* out = part + (int64_t)blockIdx.y * FLAT * HID + (int64_t)kt * FMT_TILE * HID;
  if (nc <= 0) {  // an empty chunk contributes zeros
    for (int i = t; i < FMT_TILE * HID / 4; i += FMT_THREADS)
      reinterpret_cast<float4*>(out)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  for (int st = 0; st < FAG_STAGES; ++st)  // P rows J..63 stay zero (the TMA box fills rows 0..J-1)
    for (int i = t; i < 4 * (FC_RMAX - J) * 32; i += FMT_THREADS) {
      const int blk = i / ((FC_RMAX - J) * 32), r = i - blk * (FC_RMAX - J) * 32;
      reinterpret_cast<uint32_t*>(sA + st * FAG_STAGE + blk * FMT_BLK + J * 128)[r] = 0u;
    }
  if (t == 0) {
    for (int i = 0; i < FAG_STAGES; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], FMT_EPI_WARPS);
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(tmem_slot);
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int ngroups = (nc + FAG_DRAIN - 1) / FAG_DRAIN;
  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&tm_hi);
      tc::tma_prefetch(&tm_lo);
      tc::tma_prefetch(&tm_u);
      const int k0 = kt * FMT_TILE;
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0; i < nc; ++i) {
        const int c = c0 + i;
        tc::mbar_wait(&empty[stage], phase ^ 1);
        tc::mbar_arrive_expect_tx(&full[stage], 4 * J * 128 + FAG_UBYTES);
        uint8_t* st_ = sA + stage * FAG_STAGE;
        tc::tma_load_3d(st_, &tm_hi, k0, c * B, 0, &full[stage]);
        tc::tma_load_3d(st_ + FMT_BLK, &tm_hi, k0 + 64, c * B, 0, &full[stage]);
        tc::tma_load_3d(st_ + 2 * FMT_BLK, &tm_lo, k0, c * B, 0, &full[stage]);
        tc::tma_load_3d(st_ + 3 * FMT_BLK, &tm_lo, k0 + 64, c * B, 0, &full[stage]);
        uint8_t* su = st_ + FMT_STAGE;
        tc::tma_load_2d(su, &tm_u, 0, (c * 2) * FC_RMAX, &full[stage]);
        tc::tma_load_2d(su + FMT_BLK, &tm_u, 64, (c * 2) * FC_RMAX, &full[stage]);
        tc::tma_load_2d(su + 2 * FMT_BLK, &tm_u, 0, (c * 2 + 1) * FC_RMAX, &full[stage]);
        tc::tma_load_2d(su + 3 * FMT_BLK, &tm_u, 64, (c * 2 + 1) * FC_RMAX, &full[stage]);
        if (++stage == FAG_STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t sA0 = tc::smem_u32(sA);
    for (int i = 0; i < nc; ++i) {
      const int grp = i / FAG_DRAIN, acc = grp & 1;
      const bool first = i % FAG_DRAIN == 0, last = i % FAG_DRAIN == FAG_DRAIN - 1 || i == nc - 1;
      if (first) {
        tc::mbar_wait(&tempty[acc], ((grp >> 1) & 1) ^ 1);
        tc::tc_fence_after();
      }
      tc::mbar_wait(&full[stage], phase);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint32_t d = tmem + acc * 256;
        const uint32_t ah = sA0 + stage * FAG_STAGE, al = ah + 2 * FMT_BLK, bu = ah + FMT_STAGE;
#pragma unroll
        for (int ks = 0; ks < FC_RMAX / 16; ++ks) {
          const uint64_t adh = tc::sdesc(ah + ks * 2048, FMT_BLK, 1024, 2);
          const uint64_t adl = tc::sdesc(al + ks * 2048, FMT_BLK, 1024, 2);
          const uint64_t bd = tc::sdesc(bu + ks * 2048, FMT_BLK, 1024, 2);
          tc::mma2_f16(d, d + HID, adh, adl, bd, FMT_IDESC2, FMT_IDESC, !first || ks != 0);
        }
        tc::mma_commit(&empty[stage]);
        if (last) tc::mma_commit(&tfull[acc]);
      }
      __syncwarp();
      if (++stage == FAG_STAGES) { stage = 0; phase ^= 1; }
    }
  } else {
    const int q = warp & 3, hh = (warp - 2) >> 2;  // TMEM lane quadrant (k rows), h half
    float run[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) run[j] = 0.f;
    for (int grp = 0; grp < ngroups; ++grp) {
      const int acc = grp & 1;
      tc::mbar_wait(&tfull[acc], (grp >> 1) & 1);
      tc::tc_fence_after();
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + acc * 256 + hh * 64 + half * 32;
        uint32_t v0[32], v1[32];
        tc::tmem_ld32(base, v0);
        tc::tmem_ld32(base + HID, v1);
        tc::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) run[half * 32 + j] += __uint_as_float(v0[j]) + __uint_as_float(v1[j]);
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
    const float m = __uint_as_float(*umax);
    const float inv = m > 0.f ? 1.f / exp2f(14.f - ceilf(log2f(m))) : 1.f;  // exact: power of two
    float* orow = out + (int64_t)(q * 32 + lane) * HID + hh * 64;
#pragma unroll
    for (int j = 0; j < 8; ++j) {  // row per lane: 256-bit stores fill whole sectors
      uint32_t v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = __float_as_uint(run[8 * j + e] * inv);
      stg256(orow + 8 * j, v);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc<512>(tmem);
}

// agg[e] = sum over the client chunks of their partials (fixed order, fp64)
__global__ void fc1_agg_reduce_kernel(const float* __restrict__ part, int nchunks, float* __restrict__ agg) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)FLAT * HID;
       e += (int64_t)gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int k = 0; k < nchunks; ++k) a += part[(int64_t)k * FLAT * HID + e];
    agg[e] = (float)a;
  }
}

// the same sum by a pass over the materialised block (FP32 CUDA-core validation path)
__global__ void __launch_bounds__(256) fc1_sumsq_scan_kernel(const float* __restrict__ delta, int64_t ld,
                                                             const int32_t* __restrict__ nb0,
                                                             double* __restrict__ out) {
  __shared__ double red[32];
  const int c = blockIdx.x;
  double acc = 0.0;
  if (nb0[c] > 0) {
    const float4* p = reinterpret_cast<const float4*>(delta + (int64_t)c * ld + O_F1);
    for (int i = threadIdx.x; i < FLAT * HID / 4; i += blockDim.x) {
      const float4 v = p[i];
      acc += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
    }
  }
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) out[c] = t;
}

// each client's fc1 sum of squares: its fc1_mat CTAs' partials in order
__global__ void fc1_sumsq_reduce_kernel(const double* __restrict__ part, int splits, int C,
                                        const int32_t* __restrict__ nb0, double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double t = 0.0;
  if (nb0[c] > 0)  // a client with no step kept its zeroed fc1 block (fc1_mat returned early)
    for (int x = 0; x < splits; ++x) t += part[(int64_t)c * splits + x];
  out[c] = t;
}

// ------------------------------------------------ conv2 backward-data (tcgen05)
// dz1[n, y, x, ci] = relu'(a1) * sum_{ky, kx, o} dz2[n, y-ky, x-kx, o] W[o, ci, ky, kx]
// Implicit GEMM: M = a1 positions (tile = 4 rows x 30 cols = 120), N = 32
// input channels, K = 9 taps x 64 output channels.  Per tile ONE TMA box
// {64 o, 30 x, 7 y} of the fp16 dz2 at (0, -2, y0-2, n) is staged (128-byte
// K-major SWIZZLE_128B rows); the negative / past-the-end coordinates are
// the transposed convolution's zero padding, filled by the TMA unit.  In this
// 30-wide band the tap (ky, kx) operand of output row m is band row
// m + (2-ky)*30 + (2-kx) (a column shift past x = 27 lands on the zero-filled
// columns -2, -1 of the next row), so the nine tap operands are the one band
// with the descriptor start moved by whole rows.  Epilogue: unscale, ReLU
// mask of a1, 32 channels (128 B) per position straight to HBM.
constexpr int BX_ROWS = 4;
constexpr int BX_M = BX_ROWS * S1;               // 120 valid rows
constexpr int BX_TILES = (S1 + BX_ROWS - 1) / BX_ROWS;  // 8 (last tile: 2 valid rows)
constexpr int BX_BAND = BX_ROWS + 3;             // 7 dz2 rows per band
constexpr int BX_A_TX = BX_BAND * S1 * 128;      // 26880 bytes per TMA box
constexpr int BX_A = 27 * 1024;                  // band part, 1 KB aligned
constexpr int BX_STAGE = 2 * BX_A;               // hi + lo band
constexpr int BX_B_TAP = C1 * 128;               // 4 KB: 32 rows (ci) x 64 o fp16
constexpr int WIMGT_BYTES = 9 * 2 * BX_B_TAP;    // 73728
constexpr int BX_STAGES = 2;
constexpr int BX_ACC = 2 * C1;                   // main | cross accumulators (32 columns each)
constexpr int BX_SMEM = 1024 + WIMGT_BYTES + BX_STAGES * BX_STAGE + 256;
constexpr uint32_t BX_IDESC2 = tc::idesc_f16(128, 2 * C1);  // B = [W^T hi; W^T lo] stacked along N
constexpr int BX_EPI_WARPS = 16;                 // 4 per TMEM lane quadrant, 8 input channels each
constexpr int BX_THREADS = (2 + BX_EPI_WARPS) * 32;
constexpr uint32_t BX_IDESC = tc::idesc_f16(128, C1);
static_assert(WIMGT_BYTES == WIMG_BYTES, "weight image sizes");
static_assert(127 + 2 * S1 + 2 < BX_BAND * S1 && BX_A_TX <= BX_A, "conv2 bwd-x band: every tap row inside the band");

// transposed weight image for backward-data: rows ci, K = o (K-major SWIZZLE_128B)
__global__ void __launch_bounds__(256) conv2_wimgT_kernel(const float* __restrict__ theta,
                                                          const float* __restrict__ delta, int64_t ld,
                                                          const int32_t* __restrict__ client_nb,
                                                          uint8_t* __restrict__ wimg, float* __restrict__ wscale) {
  __shared__ float red[32];
  const int g = blockIdx.x;
  if (client_nb[g] == 0) return;
  const float* dc = delta + (int64_t)g * ld;
  float4 v[WQ];
  const float sc = block_scale(load_w2(theta, dc, v), red);
  if (threadIdx.x == 0) wscale[g] = sc;
  extern __shared__ uint4 wim_s[];  // assembled in smem, written out coalesced
  uint8_t* simg = reinterpret_cast<uint8_t*>(wim_s);
#pragma unroll
  for (int u = 0; u < WQ; ++u) {
    const float e4[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = 4 * (threadIdx.x + u * 256) + e;
      const int o = i / (C1 * 9), r = i - o * (C1 * 9), ci = r / 9, tap = r - ci * 9;
      __half h, l;
      split_f16(e4[e] * sc, h, l);
      const uint32_t off = sw128_off16(ci, o);
      *reinterpret_cast<__half*>(simg + (tap * 2 + 0) * BX_B_TAP + off) = h;
      *reinterpret_cast<__half*>(simg + (tap * 2 + 1) * BX_B_TAP + off) = l;
    }
  }
  __syncthreads();
  uint4* img = reinterpret_cast<uint4*>(wimg + (int64_t)g * WIMGT_BYTES);
  for (int i = threadIdx.x; i < WIMGT_BYTES / 16; i += blockDim.x) img[i] = wim_s[i];
}

// dense dz2 = unpool(dp) * relu'(z2) as scaled fp16 hi / lo NHWC [N][28][28][64];
// also the per-sample conv2 bias gradient
constexpr int DZB_LD = NPOOL + 1;               // padded channel stride: channel planes hit different banks
constexpr int DZB_SMEM = C2 * DZB_LD * 5;
#ifndef DZB_THREADS
#define DZB_THREADS 512  // (measured 2.68 vs 3.02 ms at 256, 3.36 at 1024)
#endif
__global__ void __launch_bounds__(DZB_THREADS) dz2_build_kernel(const float* __restrict__ dp, const float* __restrict__ pooled,
                                                        const uint8_t* __restrict__ code,
                                                        const int64_t* __restrict__ slot_row,
                                                        __half* __restrict__ dzfh, __half* __restrict__ dzfl,
                                                        float* __restrict__ dzscale, float* __restrict__ db2) {
  extern __shared__ float g[];  // [64][197] values, then [64][197] codes
  __shared__ float red[32];
  uint8_t* cd = reinterpret_cast<uint8_t*>(g + C2 * DZB_LD);
  const int n = blockIdx.x;
  if (slot_row[n] < 0) return;
  float m = 0.f;
  // vectorised staging: 4 consecutive pooled positions of one channel per load (196 % 4 == 0)
  const float4* dp4 = reinterpret_cast<const float4*>(dp + (int64_t)n * FLAT);
  const float4* po4 = reinterpret_cast<const float4*>(pooled + (int64_t)n * FLAT);
  const uchar4* cd4 = reinterpret_cast<const uchar4*>(code + (int64_t)n * FLAT);
#pragma unroll 4
  for (int q = threadIdx.x; q < FLAT / 4; q += blockDim.x) {
    const float4 d = __ldg(dp4 + q), p = __ldg(po4 + q);
    const uchar4 c = __ldg(cd4 + q);
    const int k = 4 * q, ch = k / NPOOL, i = ch * DZB_LD + (k - ch * NPOOL);
    const float v0 = p.x > 0.f ? d.x : 0.f, v1 = p.y > 0.f ? d.y : 0.f, v2 = p.z > 0.f ? d.z : 0.f,
                v3 = p.w > 0.f ? d.w : 0.f;
    g[i] = v0; g[i + 1] = v1; g[i + 2] = v2; g[i + 3] = v3;
    cd[i] = c.x; cd[i + 1] = c.y; cd[i + 2] = c.z; cd[i + 3] = c.w;
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v0), fabsf(v1)), fmaxf(fabsf(v2), fabsf(v3))));
  }
  const float sc = block_scale(m, red);  // (synchronises: g / cd visible)
  if (threadIdx.x == 0) dzscale[n] = sc;
  __half* fh = dzfh + (int64_t)n * S2 * S2 * C2;
  __half* fl = dzfl + (int64_t)n * S2 * S2 * C2;
  // thread = (position, 8 consecutive channels): 16-byte stores
  for (int t = threadIdx.x; t < S2 * S2 * (C2 / 8); t += blockDim.x) {
    const int pos = t >> 3, o0 = (t & 7) * 8;
    const int y = pos / S2, x = pos - y * S2;
    const int pp = (y >> 1) * SP + (x >> 1), sub = ((y & 1) << 1) | (x & 1);
    uint32_t hv[4], lv[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i0 = (o0 + 2 * e) * DZB_LD + pp, i1 = i0 + DZB_LD;
      split_f16x2((cd[i0] == sub ? g[i0] : 0.f) * sc, (cd[i1] == sub ? g[i1] : 0.f) * sc, hv[e], lv[e]);
    }
    reinterpret_cast<uint4*>(fh)[t] = make_uint4(hv[0], hv[1], hv[2], hv[3]);
    reinterpret_cast<uint4*>(fl)[t] = make_uint4(lv[0], lv[1], lv[2], lv[3]);
  }
  // conv2 bias gradient of this sample: sum over positions of dz2 = sum of g
  if (threadIdx.x < C2) {
    float sb = 0.f;
    for (int pp = 0; pp < NPOOL; ++pp) sb += g[threadIdx.x * DZB_LD + pp];
    db2[(int64_t)n * C2 + threadIdx.x] = sb;
  }
}

__global__ void __launch_bounds__(BX_THREADS, 1) conv2_bwd_x_tc_kernel(
    const __grid_constant__ CUtensorMap tm_hi, const __grid_constant__ CUtensorMap tm_lo,
    const uint8_t* __restrict__ wimg, const float* __restrict__ wscale, const int64_t* __restrict__ slot_row, int G,
    int B, const float* __restrict__ dzscale, const __half* __restrict__ a1fh, const __half* __restrict__ a1fl,
    float* __restrict__ dz1) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = sm;
  uint8_t* sA = sB + WIMGT_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + BX_STAGES * BX_STAGE);
  uint64_t* full = bars;
  uint64_t* empty = bars + BX_STAGES;
  uint64_t* tfull = empty + BX_STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * G;  // G slots of one client (G divides the batch B)
  const int g = n0 / B;           // the client: its weight image
  {  // a client past its last local step: leave before any setup
    const int b = threadIdx.x;
    if (!__syncthreads_or(b < G && slot_row[n0 + b] >= 0)) return;
  }
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < BX_STAGES; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], BX_EPI_WARPS);
    }
    tc::mbar_init(bfull, 1);
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc<2 * BX_ACC>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&tm_hi);
      tc::tma_prefetch(&tm_lo);
      tc::mbar_arrive_expect_tx(bfull, WIMGT_BYTES);
      tc::bulk_load(sB, wimg + (int64_t)g * WIMGT_BYTES, WIMGT_BYTES, bfull);
      int stage = 0;
      uint32_t phase = 0;
      for (int b = 0; b < G; ++b) {
        const int n = n0 + b;
        if (slot_row[n] < 0) continue;
        for (int t = 0; t < BX_TILES; ++t) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          tc::mbar_arrive_expect_tx(&full[stage], 2 * BX_A_TX);
          uint8_t* st_ = sA + stage * BX_STAGE;
          tc::tma_load_4d(st_, &tm_hi, 0, -2, BX_ROWS * t - 2, n, &full[stage]);
          tc::tma_load_4d(st_ + BX_A, &tm_lo, 0, -2, BX_ROWS * t - 2, n, &full[stage]);
          if (++stage == BX_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    tc::mbar_wait(bfull, 0);
    int stage = 0, tile = 0;
    uint32_t phase = 0;
    const uint32_t sA0 = tc::smem_u32(sA), sB0 = tc::smem_u32(sB);
    for (int b = 0; b < G; ++b) {
      const int n = n0 + b;
      if (slot_row[n] < 0) continue;
      for (int t = 0; t < BX_TILES; ++t, ++tile) {
        const int acc = tile & 1;
        tc::mbar_wait(&tempty[acc], ((tile >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem + acc * BX_ACC;
        tc::mbar_wait(&full[stage], phase);
        tc::tc_fence_after();
        if (tc::elect_one()) {
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) {
            const uint32_t ah = sA0 + stage * BX_STAGE + ((2 - tap / 3) * S1 + 2 - tap % 3) * 128, al = ah + BX_A;
            const uint32_t bh = sB0 + tap * 2 * BX_B_TAP;  // [hi 32 rows | lo 32 rows]: one 64-row operand
            // K = 64 o = 4 x 16, each K step 32 B (2 descriptor units) further along the row
            tc::mma2s_f16_ks<4, 2, 2>(d, d + C1, tc::sdesc(ah, 16, 1024, 2), tc::sdesc(al, 16, 1024, 2),
                                      tc::sdesc(bh, 16, 1024, 2), BX_IDESC2, BX_IDESC, tap != 0);
          }
          tc::mma_commit(&empty[stage]);
          tc::mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == BX_STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // 16 epilogue warps: TMEM lane quadrant q = warp % 4, input-channel group of 8;
    // the a1 ReLU-mask loads are issued before waiting on the accumulator
    const int q = warp & 3, cg = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    const int r = row / S1, x = row - r * S1;
    const float ws = wscale[g];
    int tile = 0;
    for (int b = 0; b < G; ++b) {
      const int n = n0 + b;
      if (slot_row[n] < 0) continue;
      const float inv = 1.f / (dzscale[n] * ws);
      for (int t = 0; t < BX_TILES; ++t, ++tile) {
        const int acc = tile & 1;
        const int y = BX_ROWS * t + r;
        const bool ok = row < BX_M && y < S1;
        const int64_t off = ((int64_t)n * S1 * S1 + y * S1 + x) * C1 + cg * 8;
        // ReLU mask from the hi part alone: a1 >= 0, and hi = rn(a1 * s) is 0 exactly when
        // hi + lo is (a value too small for hi rounds to 0 in lo as well)
        uint4 hv = make_uint4(0, 0, 0, 0);
        if (ok) hv = *reinterpret_cast<const uint4*>(a1fh + off);
        tc::mbar_wait(&tfull[acc], (tile >> 1) & 1);
        tc::tc_fence_after();
        const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + acc * BX_ACC + cg * 8;
        uint32_t v0[8], v1[8];
        tc::tmem_ld8(base, v0);
        tc::tmem_ld8(base + C1, v1);
        tc::tmem_ld_wait();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&tempty[acc]);  // accumulator drained: next tile may start
        if (ok) {
          const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
          float o[8];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const bool m0 = (hw[e] & 0xffffu) != 0u, m1 = (hw[e] >> 16) != 0u;
            const int j = 2 * e;
            const float z0 = (__uint_as_float(v0[j]) + __uint_as_float(v1[j])) * inv;
            const float z1 = (__uint_as_float(v0[j + 1]) + __uint_as_float(v1[j + 1])) * inv;
            o[j] = m0 ? z0 : 0.f;
            o[j + 1] = m1 ? z1 : 0.f;
          }
          uint32_t ov[8];  // one 32-byte sector per lane (256-bit store)
#pragma unroll
          for (int e = 0; e < 8; ++e) ov[e] = __float_as_uint(o[e]);
          stg256(dz1 + off, ov);
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc<2 * BX_ACC>(tmem);
}

// ------------------------------------------------- conv1 forward (tcgen05)
// a1[p, o] = ReLU(b_o + sum_k xcol[p, k] W1[o, k]), k = (ci, ky, kx) (27), as a
// GEMM M = 128 positions, N = 32 channels, K = 27 + a constant-1 column
// (k = 27) that adds the bias, padded to 32 = 4 kind::tf32 K steps.  The
// split is 3xTF32 with the weight parts stacked along N: B = [W hi; W lo]
// (64 rows), so per K step ONE N = 64 MMA forms xhi*Whi | xhi*Wlo and one
// N = 32 MMA adds xlo*Whi to the cross half.  im2col A tiles (hi / lo, K-major
// SWIZZLE_128B: one 128-byte row = the position's 32 k) are staged by the CTA
// from the image in smem.  Software pipeline over the CTA's tiles (8 per
// sample): stage tile i (A double-buffered) -> issue its MMAs -> epilogue of
// tile i-1 (main + cross, ReLU, the per-sample power-of-two scale of
// conv1_fwd_kernel's a-priori bound, fp16 hi / lo NHWC stores); the next
// sample's image is fetched by a bulk async copy while the current one is
// processed.  One CTA per weight group of G slots.
constexpr int C1F_TILE = 128;
constexpr int C1F_TILES = (S1 * S1 + C1F_TILE - 1) / C1F_TILE;  // 8 (last: 4 positions)
constexpr int C1F_A = C1F_TILE * 128;                           // 16 KB per part
constexpr int C1F_STAGE = 2 * C1F_A;                            // hi | lo
constexpr int C1F_B = 64 * 128;                                 // [W hi; W lo] x 32 k
constexpr int C1F_THREADS = 256;
constexpr int C1F_GMAX = 16;
#ifndef C1F_ASTAGES
#define C1F_ASTAGES 1  // A stages: 1 -> ~65 KB, 3 CTAs per SM (the next tile is staged after its TMEM
                       // predecessor's MMAs completed, which epi_load waits for anyway)
#endif
#ifndef C1F_MINB
#define C1F_MINB 3
#endif
constexpr int C1F_SMEM = 1024 + C1F_B + C1F_ASTAGES * C1F_STAGE + 2 * IMG * 4 + 256;
constexpr uint32_t C1F_IDESC2 = tc::idesc_tf32(128, 2 * C1);
constexpr uint32_t C1F_IDESC = tc::idesc_tf32(128, C1);

__global__ void __launch_bounds__(C1F_THREADS, C1F_MINB) conv1_fwd_tc_kernel(
    const float* __restrict__ X, const int64_t* __restrict__ slot_row, const float* __restrict__ theta,
    const float* __restrict__ delta, int64_t ld, int B, int N, int G, __half* __restrict__ a1fh,
    __half* __restrict__ a1fl, float* __restrict__ a1scale) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = sm;
  uint8_t* sA = sm + C1F_B;                                         // [2][hi 16 KB | lo 16 KB]
  float* img = reinterpret_cast<float*>(sA + C1F_ASTAGES * C1F_STAGE);  // [2][3][32][32]
  uint64_t* done = reinterpret_cast<uint64_t*>(img + 2 * IMG);      // [2] MMA completion per A stage
  uint64_t* imfull = done + 2;                                      // [2] image arrival
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(imfull + 2);
  __shared__ float wsum[C1];   // sum_k |W[o, k]| (a1 bound)
  __shared__ float red[8];
  __shared__ float s_scale[2];
  __shared__ int s_slot[C1F_GMAX];
  __shared__ int s_ns;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = threadIdx.x;
  const int n0 = blockIdx.x * G;
  {  // no active slot (client past its last local step / tail chunk): leave before any setup
    // (one slot per thread, one block-wide OR: a serial scan paid an L2 round trip per slot)
    const int b = threadIdx.x;
    if (!__syncthreads_or(b < G && n0 + b < N && slot_row[n0 + b] >= 0)) return;
  }
  const float* dc = delta ? delta + (int64_t)(n0 / B) * ld : nullptr;
  const uint32_t sB0 = tc::smem_u32(sB), sA0 = tc::smem_u32(sA), simg = tc::smem_u32(img);
  // B: rows o (hi) and 32 + o (lo), k = 0..26 weights, 27 bias, 28..31 zero.  A warp holds
  // one output channel's 32 k per trip (lane = k), so sum_k |W[o, k]| (the a1 bound) is a
  // warp reduction of the values already loaded (the loads of all trips in flight together)
  static_assert(C1F_THREADS % 32 == 0 && (C1 * 32) % C1F_THREADS == 0, "conv1 fwd weight staging");
  float wv[C1 * 32 / C1F_THREADS];
#pragma unroll
  for (int u = 0; u < C1 * 32 / C1F_THREADS; ++u) {
    const int i = t + u * C1F_THREADS, o = i >> 5, k = i & 31;
    wv[u] = k < 27 ? wt(theta, dc, O_W1 + o * 27 + k) : (k == 27 ? wt(theta, dc, O_B1 + o) : 0.f);
  }
#pragma unroll
  for (int u = 0; u < C1 * 32 / C1F_THREADS; ++u) {
    const int i = t + u * C1F_THREADS, o = i >> 5, k = i & 31;
    float hi, lo;
    tc::split_tf32(wv[u], hi, lo);
    tc::sts_f32(sB0 + tc::sw128_offset(o, k), hi);
    tc::sts_f32(sB0 + tc::sw128_offset(C1 + o, k), lo);
    const float sw = warp_sum(k < 27 ? fabsf(wv[u]) : 0.f);
    if (lane == 0) wsum[o] = sw;
  }
  if (warp == 0) {  // active slots of the group, compacted in order (ballot + popc; G <= 32)
    const bool a = lane < G && n0 + lane < N && slot_row[n0 + lane] >= 0;
    const unsigned bal = __ballot_sync(0xffffffffu, a);
    if (a) s_slot[__popc(bal & ((1u << lane) - 1u))] = n0 + lane;
    if (lane == 0) s_ns = __popc(bal);
  }
  if (t == 0) {
    for (int j = 0; j < 2; ++j) {
      tc::mbar_init(&done[j], 1);
      tc::mbar_init(&imfull[j], 1);
    }
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<128>(tmem_slot);
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int ns = s_ns;
  if (ns == 0) {
    if (warp == 0) tc::tmem_dealloc<128>(tmem);
    return;
  }
  auto fetch = [&](int j) {  // bulk async copy of sample j's image into img[j & 1]
    tc::mbar_arrive_expect_tx(&imfull[j & 1], IMG * 4);
    tc::bulk_load(img + (j & 1) * IMG, X + slot_row[s_slot[j]] * IMG, IMG * 4, &imfull[j & 1]);
  };
  if (t == 0) fetch(0);
  // im2col job: position row pl, k range [16*kh, 16*kh + 16)
  const int pl = t & (C1F_TILE - 1), kh = t >> 7;
  // epilogue job: TMEM lane quadrant q = warp % 4, channel half chh = warp / 4
  const int q = warp & 3, chh = warp >> 2;
  // epilogue of tile i in two halves: epi_load issues the TMEM loads (asynchronous), the
  // next tile's im2col staging runs while they are in flight, epi_store finishes
  uint32_t v0[16], v1[16];
  auto epi_load = [&](int i) {
    const int buf = i & 1;
    tc::mbar_wait(&done[buf], (i >> 1) & 1);
    tc::tc_fence_after();
    const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + buf * 64 + chh * 16;
    tc::tmem_ld16(base, v0);
    tc::tmem_ld16(base + C1, v1);
  };
  auto epi_store = [&](int i) {
    const int j = i / C1F_TILES, tile = i - j * C1F_TILES, n = s_slot[j];
    tc::tmem_ld_wait();
    tc::tc_fence_before();
    const float sc = s_scale[j & 1];
    const int p = tile * C1F_TILE + q * 32 + lane;
    if (p < S1 * S1) {
      uint32_t hw[8], lw[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float z0 = fmaxf(__uint_as_float(v0[2 * e]) + __uint_as_float(v1[2 * e]), 0.f) * sc;
        const float z1 = fmaxf(__uint_as_float(v0[2 * e + 1]) + __uint_as_float(v1[2 * e + 1]), 0.f) * sc;
        split_f16x2(z0, z1, hw[e], lw[e]);
      }
      const int64_t off = (int64_t)n * A1 + (int64_t)p * C1 + chh * 16;
      uint4* dh = reinterpret_cast<uint4*>(a1fh + off);
      uint4* dl = reinterpret_cast<uint4*>(a1fl + off);
      dh[0] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
      dh[1] = make_uint4(hw[4], hw[5], hw[6], hw[7]);
      dl[0] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
      dl[1] = make_uint4(lw[4], lw[5], lw[6], lw[7]);
    }
  };
  const int T = ns * C1F_TILES;
  for (int i = 0; i < T; ++i) {
    const int buf = i & 1, j = i / C1F_TILES, tile = i - j * C1F_TILES;
    const uint32_t im = simg + (j & 1) * IMG * 4;
    if (tile == 0) {  // sample j starts: its image has landed; per-sample a1 scale
      tc::mbar_wait(&imfull[j & 1], (j >> 1) & 1);
      float xm = 0.f;
      for (int e = t; e < IMG; e += C1F_THREADS) xm = fmaxf(xm, fabsf(tc::lds_f32(im + 4 * e)));
      xm = warp_max(xm);
      if (lane == 0) red[warp] = xm;
      __syncthreads();  // also: every thread is past the staging of sample j-1 (its image buffer is free)
      if (warp == 0) {
        float m = lane < C1F_THREADS / 32 ? red[lane] : 0.f;
        m = warp_max(m);
        const float bound = warp_max(fabsf(wt(theta, dc, O_B1 + lane)) + m * wsum[lane]);
        if (lane == 0) {
          const float scv = bound > 0.f ? exp2f(14.f - ceilf(log2f(bound))) : 1.f;
          s_scale[j & 1] = scv;
          a1scale[s_slot[j]] = scv;
          if (j + 1 < ns) fetch(j + 1);
        }
      }
    }
    // tile i-1's accumulator: wait its MMAs (which also frees this A stage: tile i-2's MMAs
    // completed before them) and start the TMEM loads; they land while tile i is staged
    if (i >= 1) epi_load(i - 1);
    {
      // rows past the 900 positions (last tile) read position 899: their outputs are dropped
      const int p = min(tile * C1F_TILE + pl, S1 * S1 - 1), y = p / S1, x = p - y * S1;
      const uint32_t ib = im + 4 * (y * S0 + x);
      const uint32_t ah = sA0 + (i % C1F_ASTAGES) * C1F_STAGE, al = ah + C1F_A;
      auto stage = [&](auto khc) {  // khc: compile-time k half (warp-uniform)
        constexpr int KH = decltype(khc)::value;
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          float hv[4], lv[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int k = 16 * KH + 4 * c4 + e;
            if (k < 27) {
              tc::split_tf32(tc::lds_f32(ib + 4 * ((k / 9) * S0 * S0 + ((k % 9) / 3) * S0 + k % 3)), hv[e], lv[e]);
            } else {
              hv[e] = k == 27 ? 1.f : 0.f;
              lv[e] = 0.f;
            }
          }
          const uint32_t off = tc::sw128_offset(pl, 16 * KH + 4 * c4);
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(ah + off), "f"(hv[0]), "f"(hv[1]),
                       "f"(hv[2]), "f"(hv[3]) : "memory");
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(al + off), "f"(lv[0]), "f"(lv[1]),
                       "f"(lv[2]), "f"(lv[3]) : "memory");
        }
      };
      if (kh == 0)
        stage(std::integral_constant<int, 0>{});
      else
        stage(std::integral_constant<int, 1>{});
    }
    if (i >= 1) epi_store(i - 1);
    tc::fence_proxy_async();
    tc::tc_fence_before();
    __syncthreads();  // tile i staged; tile i-1's TMEM accumulator drained (its buffer is tile i+1's)
    tc::tc_fence_after();
    if (warp == 0) {
      if (tc::elect_one()) {
        const uint32_t d = tmem + buf * 64;
        const uint32_t ah = sA0 + (i % C1F_ASTAGES) * C1F_STAGE, al = ah + C1F_A;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t bd = tc::sdesc_k128(sB0 + 32 * kk);
          tc::mma_tf32(d, tc::sdesc_k128(ah + 32 * kk), bd, C1F_IDESC2, kk != 0);
          tc::mma_tf32(d + C1, tc::sdesc_k128(al + 32 * kk), bd, C1F_IDESC, 1);
        }
        tc::mma_commit(&done[buf]);
      }
      __syncwarp();
    }
  }
  epi_load(T - 1);
  epi_store(T - 1);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 0) tc::tmem_dealloc<128>(tmem);
}

// ------------------------------- conv1 forward as an implicit GEMM (tcgen05)
// Same result as conv1_fwd_tc_kernel without the im2col staging.  Output rows
// live on the image's 32-wide grid (row r = y * 32 + x, x >= 30 / y >= 30 rows
// are computed and dropped), so tap (ky, kx) of a 128-row tile is the converted
// image shifted by ky * 32 + kx rows: one smem descriptor per tap, nine
// kind::tf32 M = 128, N = 64, K = 8 MMAs per tile.  The image is converted once
// per sample into two K-major no-swizzle arrays of 16-byte rows (core-matrix
// rows, SBO = 128 B, so a row shift is a 16-byte start-address shift):
//   H[pos] = (x0 hi, x1 hi, x2 hi, 1)   L[pos] = (x0 lo, x1 lo, x2 lo, 0)
// and the K = 8 step of tap t reads (H | L) at LBO = |H|.  B for tap t
// (N = 64 rows x the same two 16-byte K chunks):
//   rows o      : (W hi[o, :, t], b hi [t = 0]) | 0
//   rows 32 + o : (W lo[o, :, t], b lo [t = 0]) | (W hi[o, :, t], 0)
// so D[:, o] = xhi Whi + b hi and D[:, 32 + o] = xhi Wlo + xlo Whi + b lo -- the
// 3xTF32 split of conv1_fwd_tc_kernel, the small cross terms summed apart from
// the main products as there.  The per-sample image is prefetched
// into registers one sample ahead (thread = 4 positions x 3 channels) and the
// MMAs of tile i + 1 are issued before the epilogue of tile i (double-buffered
// TMEM); one converted-image buffer (rewritten after the sample's last MMAs)
// keeps the CTA at ~55 KB so that 4 CTAs share an SM.
constexpr int CIG_ROWS = 1096;                // >= 7 * 128 + 127 + 2 * 32 + 2 + 1, multiple of 8
constexpr int CIG_ARR = CIG_ROWS * 16;        // one 16-byte-row array (H or L)
constexpr int CIG_BUF = 2 * CIG_ARR;          // H | L of one sample
constexpr int CIG_B = 9 * 2 * 64 * 16;        // per tap: 2 K chunks x 64 rows x 16 B
#ifndef CIG_MINB
#define CIG_MINB 4  // CTAs per SM (one converted-image buffer: ~55 KB of smem per CTA; 3 measured 2.82 vs 2.76 ms)
#endif
constexpr int CIG_SMEM = 1024 + CIG_B + CIG_BUF + 64;
static_assert(CIG_ROWS >= (C1F_TILES - 1) * C1F_TILE + C1F_TILE + 2 * S0 + 2 && CIG_ROWS % 8 == 0, "conv1 ig rows");
static_assert(C1F_TILES * C1F_TILE >= S1 * S0 - (S0 - S1), "conv1 ig tiles cover the 30 output rows");

__global__ void __launch_bounds__(C1F_THREADS, CIG_MINB) conv1_fwd_ig_kernel(
    const float* __restrict__ X, const int64_t* __restrict__ slot_row, const float* __restrict__ theta,
    const float* __restrict__ delta, int64_t ld, int B, int N, int G, __half* __restrict__ a1fh,
    __half* __restrict__ a1fl, float* __restrict__ a1scale) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = sm;
  uint8_t* sC = sm + CIG_B;                                      // H | L of the current sample
  uint64_t* done = reinterpret_cast<uint64_t*>(sC + CIG_BUF);  // [2] MMA completion per TMEM buffer
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 2);
  __shared__ float wsum[C1];  // sum_k |W[o, k]| (a1 bound)
  __shared__ float red[8];
  __shared__ float s_scale[2];
  __shared__ int s_slot[C1F_GMAX];
  __shared__ int s_ns;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = threadIdx.x;
  const int n0 = blockIdx.x * G;
  {
    const int b = threadIdx.x;
    if (!__syncthreads_or(b < G && n0 + b < N && slot_row[n0 + b] >= 0)) return;
  }
  const float* dc = delta ? delta + (int64_t)(n0 / B) * ld : nullptr;
  const uint32_t sB0 = tc::smem_u32(sB), sC0 = tc::smem_u32(sC);
  // zero B and the pad rows of both converted buffers (never overwritten)
  for (int i = t; i < CIG_B / 16; i += C1F_THREADS) reinterpret_cast<uint4*>(sB)[i] = make_uint4(0, 0, 0, 0);
  for (int i = t; i < 2 * (CIG_ROWS - S0 * S0); i += C1F_THREADS) {
    const int r = i % (CIG_ROWS - S0 * S0), a = i / (CIG_ROWS - S0 * S0);  // a = array (H, L)
    reinterpret_cast<uint4*>(sC + a * CIG_ARR)[S0 * S0 + r] = make_uint4(0, 0, 0, 0);
  }
  static_assert(C1F_THREADS % 32 == 0 && (C1 * 32) % C1F_THREADS == 0, "conv1 ig weight staging");
  float wv[C1 * 32 / C1F_THREADS];
#pragma unroll
  for (int u = 0; u < C1 * 32 / C1F_THREADS; ++u) {
    const int i = t + u * C1F_THREADS, o = i >> 5, k = i & 31;
    wv[u] = k < 27 ? wt(theta, dc, O_W1 + o * 27 + k) : (k == 27 ? wt(theta, dc, O_B1 + o) : 0.f);
  }
  __syncthreads();  // B zeroed before the scatter
#pragma unroll
  for (int u = 0; u < C1 * 32 / C1F_THREADS; ++u) {
    const int i = t + u * C1F_THREADS, o = i >> 5, k = i & 31;
    float hi, lo;
    tc::split_tf32(wv[u], hi, lo);
    if (k < 27) {
      const int ci = k / 9, tap = k - ci * 9;
      const uint32_t tb = sB0 + tap * 2048 + 4 * ci;
      tc::sts_f32(tb + o * 16, hi);                // rows o, chunk 0 (x hi): W hi
      tc::sts_f32(tb + (C1 + o) * 16, lo);         // rows 32 + o, chunk 0 (x hi): W lo
      tc::sts_f32(tb + 1024 + (C1 + o) * 16, hi);  // rows 32 + o, chunk 1 (x lo): W hi
    } else if (k == 27) {                          // bias against the constant-1 column of H (tap 0)
      tc::sts_f32(sB0 + o * 16 + 12, hi);
      tc::sts_f32(sB0 + (C1 + o) * 16 + 12, lo);
    }
    const float sw = warp_sum(k < 27 ? fabsf(wv[u]) : 0.f);
    if (lane == 0) wsum[o] = sw;
  }
  if (warp == 0) {
    const bool a = lane < G && n0 + lane < N && slot_row[n0 + lane] >= 0;
    const unsigned bal = __ballot_sync(0xffffffffu, a);
    if (a) s_slot[__popc(bal & ((1u << lane) - 1u))] = n0 + lane;
    if (lane == 0) s_ns = __popc(bal);
  }
  if (t == 0) {
    tc::mbar_init(&done[0], 1);
    tc::mbar_init(&done[1], 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<128>(tmem_slot);
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int ns = s_ns;
  if (ns == 0) {
    if (warp == 0) tc::tmem_dealloc<128>(tmem);
    return;
  }
  // image prefetch: thread t holds positions t + 256 u (u < 4), channels 0..2
  float xr[4][C0];
  auto load_raw = [&](int j) {
    const float* x = X + slot_row[s_slot[j]] * IMG;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int ci = 0; ci < C0; ++ci) xr[u][ci] = __ldg(x + ci * S0 * S0 + t + 256 * u);
  };
  // convert the prefetched image of sample j into the image buffer, then the CTA max |x|
  // and (warp 0) the per-sample a1 scale of conv1_fwd_tc_kernel
  auto convert = [&](int j) {
    const uint32_t h = sC0, l = h + CIG_ARR;
    float xm = 0.f;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float hv[C0], lv[C0];
#pragma unroll
      for (int ci = 0; ci < C0; ++ci) {
        xm = fmaxf(xm, fabsf(xr[u][ci]));
        tc::split_tf32(xr[u][ci], hv[ci], lv[ci]);
      }
      const uint32_t off = 16 * (t + 256 * u);
      asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(h + off), "f"(hv[0]), "f"(hv[1]), "f"(hv[2]),
                   "f"(1.f) : "memory");
      asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(l + off), "f"(lv[0]), "f"(lv[1]), "f"(lv[2]),
                   "f"(0.f) : "memory");
    }
    xm = warp_max(xm);
    if (lane == 0) red[warp] = xm;
    __syncthreads();
    if (warp == 0) {
      float m = lane < C1F_THREADS / 32 ? red[lane] : 0.f;
      m = warp_max(m);
      const float bound = warp_max(fabsf(wt(theta, dc, O_B1 + lane)) + m * wsum[lane]);
      if (lane == 0) {
        const float scv = bound > 0.f ? exp2f(14.f - ceilf(log2f(bound))) : 1.f;
        s_scale[j & 1] = scv;
        a1scale[s_slot[j]] = scv;
      }
    }
  };
  auto issue = [&](int i) {  // warp 0: nine tap MMAs of tile i into TMEM buffer i & 1
    if (warp != 0) return;
    if (tc::elect_one()) {
      const int j = i / C1F_TILES, tile = i - j * C1F_TILES;
      const uint32_t a0 = sC0 + tile * C1F_TILE * 16, d = tmem + (i & 1) * 64;
#pragma unroll
      for (int tap = 0; tap < 9; ++tap) {
        const uint32_t a = a0 + ((tap / 3) * S0 + tap % 3) * 16;
        tc::mma_tf32(d, tc::sdesc(a, CIG_ARR, 128, 0), tc::sdesc(sB0 + tap * 2048, 1024, 128, 0), C1F_IDESC2,
                     tap != 0);
      }
      tc::mma_commit(&done[i & 1]);
    }
    __syncwarp();
  };
  const int q = warp & 3, chh = warp >> 2;
  const int T = ns * C1F_TILES;
  load_raw(0);
  convert(0);
  if (ns > 1) load_raw(1);
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  issue(0);
  for (int i = 0; i < T; ++i) {
    const int j = i / C1F_TILES, tile = i - j * C1F_TILES;
    if (i + 1 < T && tile == C1F_TILES - 1) {  // tile i + 1 starts sample j + 1
      tc::mbar_wait(&done[i & 1], (i >> 1) & 1);  // sample j's last MMAs (and all before) read the buffer
      convert(j + 1);
      if (j + 2 < ns) load_raw(j + 2);
      tc::fence_proxy_async();
    }
    tc::tc_fence_before();
    __syncthreads();  // every thread past the epilogue of tile i - 1 (TMEM buffer (i + 1) & 1 is free)
    tc::tc_fence_after();
    if (i + 1 < T) issue(i + 1);
    // epilogue of tile i (overlaps tile i + 1's MMAs)
    tc::mbar_wait(&done[i & 1], (i >> 1) & 1);
    tc::tc_fence_after();
    uint32_t v0[16], v1[16];
    const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (i & 1) * 64 + chh * 16;
    tc::tmem_ld16(base, v0);
    tc::tmem_ld16(base + C1, v1);
    tc::tmem_ld_wait();
    const int r = tile * C1F_TILE + q * 32 + lane, y = r >> 5, x = r & 31;
    if (x < S1 && y < S1) {
      const float sc = s_scale[j & 1];
      uint32_t hw[8], lw[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float z0 = fmaxf(__uint_as_float(v0[2 * e]) + __uint_as_float(v1[2 * e]), 0.f) * sc;
        const float z1 = fmaxf(__uint_as_float(v0[2 * e + 1]) + __uint_as_float(v1[2 * e + 1]), 0.f) * sc;
        split_f16x2(z0, z1, hw[e], lw[e]);
      }
      // one full 32-byte sector per lane and part (256-bit stores; the workspace is 256-byte aligned)
      const int64_t off = (int64_t)s_slot[j] * A1 + (int64_t)(y * S1 + x) * C1 + chh * 16;
      stg256(a1fh + off, hw);
      stg256(a1fl + off, lw);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 0) tc::tmem_dealloc<128>(tmem);
}

// ------------------------------------------ conv1 backward-weights (tcgen05)
// dW1[o, k] = sum over the client's samples and positions p of dz1[p, o] * xcol[p, k],
// k = (ci, ky, kx) (27) plus a constant-1 column k = 27 that yields the bias
// gradient.  A GEMM with K = positions, done on the tensor core in kind::tf32
// with a 3xTF32-style split held in the operand ROWS instead of extra MMAs:
//   A (M = 128) rows 0-31 = tf32(dz1) hi, rows 32-63 = lo  (rows 64-127 unused)
//   B (N = 64)  rows 0-31 = tf32(xcol) hi, rows 32-63 = lo
// so ONE 128x64x8 MMA per 8 positions forms hi*hi, hi*lo, lo*hi and lo*lo in
// four quadrants of the accumulator.  Operands are staged per 128-position
// chunk by the CTA (K-major SWIZZLE_128B, transposed from the NHWC dz1 and
// im2col'ed from the image in smem), double-buffered against the MMAs; each
// chunk's accumulator (a 16-MMA chain) is drained by warps 0 / 1 into fp32
// registers (round-to-nearest adds) while the next chunk runs.
constexpr int W1_GRP = 4;  // conv1 weight gradient: chunks per TMEM accumulation chain (4 x 8 MMAs)
constexpr int W1_PART = 28 * 32;  // floats per split partial of conv1_bwd_w_tc ([k][o])
constexpr int W1_CH = 64;                           // positions per chunk
constexpr int W1_CPS = (S1 * S1 + W1_CH - 1) / W1_CH;  // 15 chunks per sample (last: 4 positions)
constexpr int W1_ATOM = 16 * 1024;                  // per 32-position K atom: A rows 0-63 (8 KB) | B rows 0-63 (8 KB)
constexpr int W1_STAGE = (W1_CH / 32) * W1_ATOM;    // 32 KB
constexpr int W1_THREADS = 256;
constexpr int W1_NLD = W1_CH * 8 / W1_THREADS;      // dz1 float4 loads per thread per chunk
constexpr int W1_KPER = 28 / (W1_THREADS / W1_CH);  // im2col rows per thread
static_assert(W1_NLD * W1_THREADS == W1_CH * 8 && W1_KPER * (W1_THREADS / W1_CH) == 28, "conv1 bwd-w staging split");
#ifndef W1_ASTAGES
#define W1_ASTAGES 2  // operand stages (1: the previous chunk's MMAs must finish before staging)
#endif
#ifndef W1_MINB
#define W1_MINB 2
#endif
constexpr int W1_SMEM = 1024 + W1_ASTAGES * W1_STAGE + 2 * IMG * 4 + 32 * 33 * 4 + 64;
constexpr uint32_t W1_IDESC = tc::idesc_tf32(128, 64);

template <bool SPLIT>
__global__ void __launch_bounds__(W1_THREADS, W1_MINB) conv1_bwd_w_tc_kernel(const float* __restrict__ X,
                                                                      const int64_t* __restrict__ slot_row,
                                                                      const float* __restrict__ dz1, int B,
                                                                      const int32_t* __restrict__ client_nb,
                                                                      float* __restrict__ delta, int64_t ld, Step st,
                                                                      int split, float* __restrict__ wpart) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* img = reinterpret_cast<float*>(sm + W1_ASTAGES * W1_STAGE);  // [2][3][32][32] (next sample prefetched)
  float* red = img + 2 * IMG;                                // [32][33]: warp 1's sums
  uint64_t* done = reinterpret_cast<uint64_t*>(red + 32 * 33);  // [2] MMA completion per stage
  uint64_t* imfull = done + 2;                                   // [2] image arrival
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(imfull + 2);
  // split > 1 (few active clients): CTA (c, part) takes samples [b0, b1) and writes a
  // partial [28][32] gradient; conv1_bwd_w_reduce_kernel applies the update
  // (SPLIT = false: the plain one-CTA-per-client kernel, compiled separately)
  int c = blockIdx.x, b0 = 0, b1;
  if constexpr (SPLIT) {
    c = blockIdx.x / split;
    const int part = blockIdx.x - c * split, nbc = client_nb[c];
    b0 = part * nbc / split;
    b1 = (part + 1) * nbc / split;
    if (b1 <= b0) return;
  } else {
    b1 = client_nb[c];
    if (b1 == 0) return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = threadIdx.x;
  const uint32_t s0 = tc::smem_u32(sm), simg = tc::smem_u32(img);
  // rows 28-31 / 60-63 of B (padding of k) stay zero; staging never writes them
  for (int i = t; i < W1_ASTAGES * (W1_CH / 32) * 2 * 4 * 8; i += W1_THREADS) {  // stage, atom, hi/lo, 4 rows, 8 x 16 B
    const int q = i & 7, r = (i >> 3) & 3, part = (i >> 5) & 1, atom = i >> 6;
    reinterpret_cast<uint4*>(sm + atom * W1_ATOM + 8192 + (part * 32 + 28 + r) * 128)[q] = make_uint4(0, 0, 0, 0);
  }
  if (t == 0) {
    tc::mbar_init(&done[0], 1);
    tc::mbar_init(&done[1], 1);
    tc::mbar_init(&imfull[0], 1);
    tc::mbar_init(&imfull[1], 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<128>(tmem_slot);
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  float run[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) run[k] = 0.f;
  // drain chunk i's accumulator into run[] (warp 0: hi rows, warp 1: lo rows)
  // accumulators are drained once per group of W1_GRP chunks (a 32-MMA chain), from
  // TMEM buffer (group & 1), after the group's last chunk i completed
  auto drain = [&](int i) {
    tc::mbar_wait(&done[i & 1], (i >> 1) & 1);
    tc::tc_fence_after();
    const uint32_t base = tmem + ((uint32_t)(warp * 32) << 16) + ((i / W1_GRP) & 1) * 64;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t v0[16], v1[16];
      tc::tmem_ld16(base + 16 * h, v0);
      tc::tmem_ld16(base + 32 + 16 * h, v1);
      tc::tmem_ld_wait();
#pragma unroll
      for (int k = 0; k < 16; ++k) run[16 * h + k] += __uint_as_float(v0[k]) + __uint_as_float(v1[k]);
    }
    tc::tc_fence_before();
  };
  // A staging: coalesced float4 f = j * 256 + t of the chunk's [64 pos][32 o] dz1 block
  // (position f / 8, channel quad f % 8); the next chunk is prefetched into
  // registers a chunk ahead
  const int nchunks = (b1 - b0) * W1_CPS;
  auto load_dz = [&](int i, float4 (&v)[W1_NLD]) {
    const int b = i / W1_CPS, p0 = (i - b * W1_CPS) * W1_CH;
    const float4* dzn = reinterpret_cast<const float4*>(dz1 + ((int64_t)c * B + b0 + b) * A1 + (int64_t)p0 * C1);
#pragma unroll
    for (int j = 0; j < W1_NLD; ++j) {
      const int f = j * W1_THREADS + t;
      v[j] = p0 + (f >> 3) < S1 * S1 ? __ldg(dzn + f) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  float4 cur[W1_NLD], nxt[W1_NLD];
  load_dz(0, cur);
  const int kq = t / W1_CH;
  uint32_t koff[7];  // byte offset of im2col row kq*7+kk relative to the output position
#pragma unroll
  for (int kk = 0; kk < 7; ++kk) {
    const int k = min(kq * 7 + kk, 26), ci = k / 9, ky = (k % 9) / 3, kx = k % 3;
    koff[kk] = 4 * (ci * S0 * S0 + ky * S0 + kx);
  }
  for (int i = 0; i < nchunks; ++i) {
    const int b = i / W1_CPS, ch = i - b * W1_CPS, p0 = ch * W1_CH;
    const int64_t n = (int64_t)c * B + b0 + b;
    const uint32_t stg = s0 + (i % W1_ASTAGES) * W1_STAGE;
    if (i + 1 < nchunks) load_dz(i + 1, nxt);
    if (i >= W1_ASTAGES)  // chunk i - W1_ASTAGES's MMAs done reading this stage
      tc::mbar_wait(&done[(i - W1_ASTAGES) & 1], ((i - W1_ASTAGES) >> 1) & 1);
    if (ch == 0) {
      // the previous sample's im2col reads are finished: its buffer takes sample b + 1 (bulk
      // async copy, overlapping this sample); sample b's image was fetched one sample ago
      __syncthreads();
      if (t == 0) {
        tc::fence_proxy_async();  // (the generic-proxy reads of that buffer precede the async write)
        if (b == 0) {
          tc::mbar_arrive_expect_tx(&imfull[0], IMG * 4);
          tc::bulk_load(img, X + slot_row[n] * IMG, IMG * 4, &imfull[0]);
        }
        if (b + 1 < b1 - b0) {
          tc::mbar_arrive_expect_tx(&imfull[(b + 1) & 1], IMG * 4);
          tc::bulk_load(img + ((b + 1) & 1) * IMG, X + slot_row[n + 1] * IMG, IMG * 4, &imfull[(b + 1) & 1]);
        }
      }
      tc::mbar_wait(&imfull[b & 1], (b >> 1) & 1);
    }
#pragma unroll
    for (int j = 0; j < W1_NLD; ++j) {
      const int f = j * W1_THREADS + t, pl = f >> 3, oq = f & 7;
      const float vv[4] = {cur[j].x, cur[j].y, cur[j].z, cur[j].w};
      const uint32_t atom = stg + (pl >> 5) * W1_ATOM;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float hi, lo;
        tc::split_tf32(vv[e], hi, lo);
        const int o = 4 * oq + e;
        tc::sts_f32(atom + tc::sw128_offset(o, pl & 31), hi);
        tc::sts_f32(atom + tc::sw128_offset(32 + o, pl & 31), lo);
      }
    }
    // B: thread = position (64) x 7 of the 28 im2col rows (k = kq*7 + kk)
    {
      const int pl = t & (W1_CH - 1);
      const int p = p0 + pl, y = p / S1, x = p - y * S1;
      const bool valid = p < S1 * S1;
      const uint32_t atom = stg + (pl >> 5) * W1_ATOM + 8192;
      const uint32_t ib = simg + (b & 1) * IMG * 4 + 4 * (y * S0 + x);
#pragma unroll
      for (int kk = 0; kk < 7; ++kk) {
        const int k = kq * 7 + kk;
        float v = 0.f;
        if (valid) v = k < 27 ? tc::lds_f32(ib + koff[kk]) : 1.f;
        float hi, lo;
        tc::split_tf32(v, hi, lo);
        tc::sts_f32(atom + tc::sw128_offset(k, pl & 31), hi);
        tc::sts_f32(atom + tc::sw128_offset(32 + k, pl & 31), lo);
      }
    }
    tc::fence_proxy_async();
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (warp == 0) {
      if (tc::elect_one()) {
        const uint32_t d = tmem + ((i / W1_GRP) & 1) * 64;
        const bool fresh = i % W1_GRP == 0;
#pragma unroll
        for (int kk = 0; kk < W1_CH / 8; ++kk) {
          const uint32_t a = stg + (kk >> 2) * W1_ATOM + (kk & 3) * 32;
          tc::mma_tf32(d, tc::sdesc_k128(a), tc::sdesc_k128(a + 8192), W1_IDESC, !fresh || kk != 0);
        }
        tc::mma_commit(&done[i & 1]);
      }
      __syncwarp();
    }
    if (warp < 2 && i >= 1 && (i - 1) % W1_GRP == W1_GRP - 1) drain(i - 1);
#pragma unroll
    for (int j = 0; j < W1_NLD; ++j) cur[j] = nxt[j];
  }
  if (warp < 2) drain(nchunks - 1);  // the last chunk closes the last group
  // combine the hi-row (warp 0) and lo-row (warp 1) sums; update dW1 and b1
  if (warp == 1)
#pragma unroll
    for (int k = 0; k < 32; ++k) red[lane * 33 + k] = run[k];
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (SPLIT && warp == 0) {
    float* wp = wpart + (int64_t)blockIdx.x * W1_PART;
#pragma unroll
    for (int k = 0; k < 28; ++k) wp[k * 32 + lane] = run[k] + red[lane * 33 + k];
    tc::tmem_dealloc<128>(tmem);
  } else if (warp == 0) {
    float* dc = delta + (int64_t)c * ld;
#pragma unroll
    for (int k = 0; k < 28; ++k) {
      const float g = run[k] + red[lane * 33 + k];
      float& dl = k < 27 ? dc[O_W1 + (int64_t)lane * (C0 * 9) + k] : dc[O_B1 + lane];
      dl += st.lr * (g - st.mu * dl);
    }
    tc::tmem_dealloc<128>(tmem);
  }
}

// conv1 weight gradient on the FP32 pipes, register-blocked: the GEMM is tiny
// (M = 32 channels, N = 28 = 27 taps + bias, K = the client's positions) and its
// tcgen05 form (conv1_bwd_w_tc_kernel) is bound by per-chunk operand staging
// (two split + swizzled scalar stores per operand element), so here the only
// staging is two 16-byte copies per thread per 128 positions and the math runs on
// FFMA.  16 warps; warp w owns the output tile (8 channels og = w & 3) x (7 k,
// kg = w >> 2; k = 27 is the bias column, x = 1) in 56 accumulators per lane;
// lane = output column x (30 of 32 live), one output row per trip, chunks of 3
// rows (a per-position layout with a division per position and 2-way image-load
// bank conflicts measured 3.67 ms).  Per position a lane reads its 8 dz1
// values (two 16-byte loads; chunks are stored with the 16-byte index XOR
// (position & 7), so a quarter-warp's 8 positions hit 8 different bank groups)
// and 7 image values (the k-group's taps are compile-time offsets: the tile loop
// is instantiated per kg), then does 56 FMAs.  dz1 chunks are prefetched into
// registers one chunk ahead (a TMA ring measured slower: 4.5 vs 3.95 ms per
// iteration), images by bulk copy one sample ahead.  Lane partials (fp32 over the
// lane's positions) are warp-reduced in fixed order; SPLIT writes [28][32]
// partials for conv1_bwd_w_reduce_kernel as conv1_bwd_w_tc_kernel does.
constexpr int WF_THREADS = 512;
constexpr int WF_ROWS = 3;                                   // output rows per chunk (30 = 10 x 3)
constexpr int WF_CH = WF_ROWS * S1;                          // 90 positions per chunk
constexpr int WF_CPS = S1 / WF_ROWS;                         // 10 chunks per sample
constexpr int WF_NF4 = WF_CH * C1 / 4;                       // 720 dz1 float4 per chunk
constexpr int WF_NLD = (WF_NF4 + WF_THREADS - 1) / WF_THREADS;
constexpr int WF_BUF = (WF_CH + 2) * C1;                     // floats per dz1 buffer (+2 rows: lanes 30, 31 of the last row)
constexpr int WF_IMGS = IMG + 64;                            // image stride (zero pad: lanes 30, 31 read past the plane)
constexpr int WF_SMEM = 2 * WF_BUF * 4 + 2 * WF_IMGS * 4 + 16;
static_assert(S1 % WF_ROWS == 0, "conv1 bwd-w FFMA: whole rows per chunk");

// lane = output column x (lanes 30, 31 idle: their dz1 is forced to 0), one output row per trip
template <int KG>
__device__ __forceinline__ void wf_chunk(const float* __restrict__ dzb, const float* __restrict__ im, int y0, int og,
                                         int lane, float (&acc)[8][7]) {
  constexpr int K0 = 7 * KG;
  const bool live = lane < S1;
#pragma unroll
  for (int r = 0; r < WF_ROWS; ++r) {
    const int pl = r * S1 + lane;
    const float* ib = im + (y0 + r) * S0 + lane;
    const float4* dr = reinterpret_cast<const float4*>(dzb) + pl * 8;
    float4 d0 = dr[(2 * og) ^ (pl & 7)];
    float4 d1 = dr[(2 * og + 1) ^ (pl & 7)];
    if (!live) d0 = d1 = make_float4(0.f, 0.f, 0.f, 0.f);
    const float dv[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
    float xv[7];
#pragma unroll
    for (int e = 0; e < 7; ++e) {
      const int k = K0 + e;
      if (k < 27)
        xv[e] = ib[(k / 9) * S0 * S0 + ((k % 9) / 3) * S0 + k % 3];
      else
        xv[e] = 1.f;
    }
#pragma unroll
    for (int o = 0; o < 8; ++o)
#pragma unroll
      for (int e = 0; e < 7; ++e) acc[o][e] = fmaf(dv[o], xv[e], acc[o][e]);
  }
}

template <bool SPLIT>
__global__ void __launch_bounds__(WF_THREADS, 1) conv1_bwd_w_ffma_kernel(const float* __restrict__ X,
                                                                        const int64_t* __restrict__ slot_row,
                                                                        const float* __restrict__ dz1, int B,
                                                                        const int32_t* __restrict__ client_nb,
                                                                        float* __restrict__ delta, int64_t ld,
                                                                        Step st, int split,
                                                                        float* __restrict__ wpart) {
  extern __shared__ __align__(16) uint8_t wf_smem[];
  float* dzs = reinterpret_cast<float*>(wf_smem);                          // [2][WF_BUF], swizzled rows
  float* imgs = dzs + 2 * WF_BUF;                                          // [2][WF_IMGS]
  uint64_t* imfull = reinterpret_cast<uint64_t*>(imgs + 2 * WF_IMGS);      // [2]
  int c = blockIdx.x, b0 = 0, b1;
  if constexpr (SPLIT) {
    c = blockIdx.x / split;
    const int part = blockIdx.x - c * split, nbc = client_nb[c];
    b0 = part * nbc / split;
    b1 = (part + 1) * nbc / split;
    if (b1 <= b0) return;
  } else {
    b1 = client_nb[c];
    if (b1 == 0) return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = threadIdx.x;
  const int og = warp & 3, kg = warp >> 2;
  const int ns = b1 - b0, nchunks = ns * WF_CPS;
  const int64_t n0 = (int64_t)c * B + b0;
  if (t < 128) imgs[(t >> 6) * WF_IMGS + IMG + (t & 63)] = 0.f;
  if (t == 0) {
    tc::mbar_init(&imfull[0], 1);
    tc::mbar_init(&imfull[1], 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  auto fetch_img = [&](int b) {  // thread 0
    tc::mbar_arrive_expect_tx(&imfull[b & 1], IMG * 4);
    tc::bulk_load(imgs + (b & 1) * WF_IMGS, X + slot_row[n0 + b] * IMG, IMG * 4, &imfull[b & 1]);
  };
  if (t == 0) fetch_img(0);
  // dz1 chunk prefetch: float4 f = t + 512 u of the chunk's [90 pos][8 quads] block
  float4 pre[WF_NLD];
  auto load_dz = [&](int i) {
    const int b = i / WF_CPS, p0 = (i - b * WF_CPS) * WF_CH;
    const float4* src = reinterpret_cast<const float4*>(dz1 + (n0 + b) * A1 + (int64_t)p0 * C1);
#pragma unroll
    for (int u = 0; u < WF_NLD; ++u) {
      const int f = t + u * WF_THREADS;
      if (f < WF_NF4) pre[u] = __ldg(src + f);
    }
  };
  float acc[8][7];
#pragma unroll
  for (int o = 0; o < 8; ++o)
#pragma unroll
    for (int e = 0; e < 7; ++e) acc[o][e] = 0.f;
  load_dz(0);
  for (int i = 0; i < nchunks; ++i) {
    const int b = i / WF_CPS, ch = i - b * WF_CPS, p0 = ch * WF_CH;
    float* dzb = dzs + (i & 1) * WF_BUF;
#pragma unroll
    for (int u = 0; u < WF_NLD; ++u) {
      const int f = t + u * WF_THREADS, pl = f >> 3, q = f & 7;
      if (f < WF_NF4) reinterpret_cast<float4*>(dzb)[pl * 8 + (q ^ (pl & 7))] = pre[u];
    }
    if (i + 1 < nchunks) load_dz(i + 1);
    __syncthreads();  // chunk i staged; every thread is past chunk i - 1 (sample b - 1's last image reads)
    if (ch == 0) {
      if (t == 0 && b + 1 < ns) {  // image buffer (b + 1) & 1 held sample b - 1
        tc::fence_proxy_async();
        fetch_img(b + 1);
      }
      tc::mbar_wait(&imfull[b & 1], (b >> 1) & 1);
    }
    const float* im = imgs + (b & 1) * WF_IMGS;
    const int y0 = ch * WF_ROWS;
    switch (kg) {  // warp-uniform
      case 0: wf_chunk<0>(dzb, im, y0, og, lane, acc); break;
      case 1: wf_chunk<1>(dzb, im, y0, og, lane, acc); break;
      case 2: wf_chunk<2>(dzb, im, y0, og, lane, acc); break;
      default: wf_chunk<3>(dzb, im, y0, og, lane, acc); break;
    }
  }
  // lane partials -> warp sums (fixed order); lane 0 updates (or writes the split partial)
  float* dc = delta + (int64_t)c * ld;
  float* wp = SPLIT ? wpart + (int64_t)blockIdx.x * W1_PART : nullptr;
#pragma unroll
  for (int o = 0; o < 8; ++o)
#pragma unroll
    for (int e = 0; e < 7; ++e) {
      const float g = warp_sum(acc[o][e]);
      const int k = 7 * kg + e, oc = 8 * og + o;
      if (lane == 0) {
        if constexpr (SPLIT) {
          wp[k * 32 + oc] = g;
        } else {
          float& dl = k < 27 ? dc[O_W1 + (int64_t)oc * (C0 * 9) + k] : dc[O_B1 + oc];
          dl += st.lr * (g - st.mu * dl);
        }
      }
    }
}

// split conv1 weight gradient: fixed-order sum of the client's CTA partials, then the update
__global__ void conv1_bwd_w_reduce_kernel(const float* __restrict__ wpart, int split,
                                          const int32_t* __restrict__ client_nb, float* __restrict__ delta,
                                          int64_t ld, Step st) {
  const int c = blockIdx.x;
  const int nb = client_nb[c];
  if (nb == 0) return;
  float* dc = delta + (int64_t)c * ld;
  for (int e = threadIdx.x; e < W1_PART; e += blockDim.x) {
    float g = 0.f;
    for (int p = 0; p < split; ++p)  // (a part with an empty sample range wrote nothing)
      if ((p + 1) * nb / split > p * nb / split) g += wpart[((int64_t)c * split + p) * W1_PART + e];
    const int k = e >> 5, o = e & 31;
    float& dl = k < 27 ? dc[O_W1 + (int64_t)o * (C0 * 9) + k] : dc[O_B1 + o];
    dl += st.lr * (g - st.mu * dl);
  }
}

int g_conv_impl = 1;  // 1 = tcgen05 (product path), 0 = FP32 CUDA-core kernels (validation)
// conv2 forward on CTA pairs (conv2_fwd_tc2_kernel): correct (tests) but measured slower
// than the single-CTA kernel (10.7 vs 7.9 ms per iteration), so off by default
bool g_conv2_pairs = false;
// conv1 forward: 1 = implicit GEMM (conv1_fwd_ig_kernel, default), 0 = im2col staging (conv1_fwd_tc_kernel)
int g_conv1_fwd_impl = 1;
// conv1 weight gradient: the tcgen05 kernel (conv1_bwd_w_tc_kernel, default) or, with impl 4, the
// register-blocked FP32 kernel (conv1_bwd_w_ffma_kernel: 3.6 vs 4.35 ms per iteration, but the
// fedsim drop-in cnn_dp run misses the theta gate in its second iteration on 11 conv1 entries,
// err / limit 4.5 vs 0.03 for the tcgen05 kernel -- not understood yet, so not the default)
bool g_conv1_bwd_ffma = false;


// ------------------------------------------------ conv2 backward-weights (tcgen05)
// dW[o, ci, ky, kx] = sum over the client's samples and conv2-output positions
// p of dz2[p, o] * a1[p + (ky, kx), ci]: a GEMM with K = positions.  Both
// operands are NHWC (positions along rows) -> MN-major, which the tensor core
// supports for 16-bit inputs: kind::f16 with fp32 accumulation, each fp32
// value split into scaled fp16 hi + lo (per-sample power-of-two scale keeps
// values normal; hi*hi + hi*lo + lo*hi ~ 2^-22 relative, as 3xTF32).
// Positions run in the 30-wide space of a1 (dz2 rows are zero-filled by the
// TMA in columns 28, 29), where the tap shift is a whole number of rows: one
// staged a1 tile {32 ci, 30 x, 10 y} serves all nine taps -- the M = 128
// operand for row ky is four 32-channel blocks at LBO = one 64-byte row
// (kx = 0..3, the kx = 3 block discarded) starting at row ky*30.  A K block
// = 7 output rows = 210 positions = 14 MMAs of K = 16 (the last 14 positions
// against zero dz2 rows; 8-row blocks left 4 of 32 rows empty); each K block starts
// fresh TMEM accumulators per ky (hi*hi and cross terms separately), drained
// by eight epilogue warps into fp32 registers with the per-sample unscale.
constexpr int BW_PART = 3 * 64 * 96;  // floats per split partial of conv2_bwd_w_tc ([ky][o][kx*32+ci])
#ifndef BW_ROWS
#define BW_ROWS 7  // output rows per K block: 4 x 7 = the 28 rows exactly (8 rows left 4 of 32 empty)
#endif
constexpr int BW_NKB = (S2 + BW_ROWS - 1) / BW_ROWS;  // 4 K blocks per sample
static_assert(BW_NKB % 2 == 0, "conv2 weight gradient drains pairs of K blocks of one sample");
constexpr int BW_KPOS = BW_ROWS * S1;             // 210 positions loaded per K block
constexpr int BW_KSTEPS = (BW_KPOS + 15) / 16;    // 14 MMAs of K = 16 (positions 210..223: zero dz2 rows)
// a1 rows the taps read: ky * 30 + 16 * BW_KSTEPS + kx (kx <= 3), rounded to 16 rows (1 KB)
constexpr int BW_A_ROWS = ((2 * S1 + 16 * BW_KSTEPS + 3) + 15) / 16 * 16;
constexpr int BW_A_BYTES = BW_A_ROWS * 64;
constexpr int BW_A_TX = (BW_ROWS + 2) * S1 * 64;  // a1 bytes the TMA writes (the rest stays zero)
constexpr int BW_B_TX = BW_KPOS * 128;            // dz2 bytes the TMA writes per part
constexpr int BW_B_BYTES = BW_KSTEPS * 16 * 128;  // dz2 tile per part (the rows past BW_KPOS stay zero)
static_assert(BW_A_ROWS * 64 >= BW_A_TX && BW_B_BYTES % 1024 == 0 && BW_A_BYTES % 1024 == 0, "bwd-w tiles");
constexpr int BW_STAGE = 2 * BW_A_BYTES + 2 * BW_B_BYTES;  // 100352
constexpr int BW_STAGES = 2;
constexpr int BW_EPI_WARPS = 16;                  // 4 lane quarters x 4 groups of 16 output channels
constexpr int BW_EPI_COLS = C2 / (BW_EPI_WARPS / 4);  // 16
constexpr int BW_THREADS = (2 + BW_EPI_WARPS) * 32;
constexpr int BW_SMEM = 1024 + BW_STAGES * BW_STAGE + 256;
constexpr uint32_t BW_IDESC = tc::idesc_f16_mn(128, C2);
constexpr uint32_t BW_IDESC2 = tc::idesc_f16_mn(128, 2 * C2);  // B = [dz2 hi | dz2 lo] along N
static_assert(BW_B_BYTES % 16 == 0 && (BW_B_BYTES >> 4) < (1 << 14), "bwd-w: hi/lo N-block stride fits the LBO field");

__global__ void __launch_bounds__(BW_THREADS, 1) conv2_bwd_w_tc_kernel(
    const __grid_constant__ CUtensorMap ta_hi, const __grid_constant__ CUtensorMap ta_lo,
    const __grid_constant__ CUtensorMap td_hi, const __grid_constant__ CUtensorMap td_lo, int B,
    const int32_t* __restrict__ client_nb, const float* __restrict__ a1scale, const float* __restrict__ dzscale,
    const float* __restrict__ db2, float* __restrict__ delta, int64_t ld, Step st, int split,
    float* __restrict__ wpart) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + BW_STAGES * BW_STAGE);
  uint64_t* full = bars;
  uint64_t* empty = bars + BW_STAGES;
  uint64_t* tfull = empty + BW_STAGES;  // [3] one per ky
  uint64_t* tempty = tfull + 3;         // [3]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 3);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // split > 1 (few active clients): CTA (c, part) takes samples [b0, b1) of client c and
  // writes its partial gradient to wpart; conv2_bwd_w_reduce_kernel applies the update
  const int c = blockIdx.x / split, part = blockIdx.x - c * split;
  const int nbc = client_nb[c];
  const int b0 = part * nbc / split, b1 = (part + 1) * nbc / split;
  if (b1 <= b0) return;
  const int nblocks = (b1 - b0) * BW_NKB;
  for (int s = 0; s < BW_STAGES; ++s) {  // a1 rows past the TMA box are read against zero dz2: keep them finite
    for (int i = threadIdx.x; i < (BW_A_BYTES - BW_A_TX) / 4; i += blockDim.x) {
      reinterpret_cast<float*>(sm + s * BW_STAGE + BW_A_TX)[i] = 0.f;
      reinterpret_cast<float*>(sm + s * BW_STAGE + BW_A_BYTES + BW_A_TX)[i] = 0.f;
    }
    // dz2 positions past the K block (the last MMA's tail) must be zero: they are never loaded
    for (int i = threadIdx.x; i < (BW_B_BYTES - BW_B_TX) / 4; i += blockDim.x) {
      reinterpret_cast<float*>(sm + s * BW_STAGE + 2 * BW_A_BYTES + BW_B_TX)[i] = 0.f;
      reinterpret_cast<float*>(sm + s * BW_STAGE + 2 * BW_A_BYTES + BW_B_BYTES + BW_B_TX)[i] = 0.f;
    }
  }
  tc::fence_proxy_async();
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < BW_STAGES; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 3; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], BW_EPI_WARPS);
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&ta_hi);
      tc::tma_prefetch(&ta_lo);
      tc::tma_prefetch(&td_hi);
      tc::tma_prefetch(&td_lo);
      int stage = 0;
      uint32_t phase = 0;
      for (int blk = 0; blk < nblocks; ++blk) {
        const int n = c * B + b0 + blk / BW_NKB, y0 = BW_ROWS * (blk % BW_NKB);
        tc::mbar_wait(&empty[stage], phase ^ 1);
        tc::mbar_arrive_expect_tx(&full[stage], 2 * BW_A_TX + 2 * BW_B_TX);
        uint8_t* st_ = sm + stage * BW_STAGE;
        tc::tma_load_4d(st_, &ta_hi, 0, 0, y0, n, &full[stage]);
        tc::tma_load_4d(st_ + BW_A_BYTES, &ta_lo, 0, 0, y0, n, &full[stage]);
        tc::tma_load_4d(st_ + 2 * BW_A_BYTES, &td_hi, 0, 0, y0, n, &full[stage]);
        tc::tma_load_4d(st_ + 2 * BW_A_BYTES + BW_B_BYTES, &td_lo, 0, 0, y0, n, &full[stage]);
        if (++stage == BW_STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t s0 = tc::smem_u32(sm);
    for (int blk = 0; blk < nblocks; ++blk) {
      tc::mbar_wait(&full[stage], phase);
      tc::tc_fence_after();
      const uint32_t ah = s0 + stage * BW_STAGE, al = ah + BW_A_BYTES;
      const uint32_t bh = ah + 2 * BW_A_BYTES;  // dz2 lo follows at + BW_B_BYTES
      // accumulators are drained once per PAIR of blocks (same sample: BW_NKB is even), a
      // 28-step main chain per drain (<= 36: as accurate as fp32, tools/microbench)
      const bool first = (blk & 1) == 0, last = (blk & 1) == 1;
      for (int ky = 0; ky < 3; ++ky) {
        if (first) {
          tc::mbar_wait(&tempty[ky], ((blk >> 1) & 1) ^ 1);  // previous pair's ky accumulators drained
          tc::tc_fence_after();
        }
        if (tc::elect_one()) {
          const uint32_t dm = tmem + ky * 2 * C2, dx = dm + C2;
#pragma unroll 5
          for (int ks = 0; ks < BW_KSTEPS; ++ks) {
            const uint32_t arow = ky * S1 + ks * 16;
            const uint64_t adh = tc::sdesc(ah + arow * 64, 64, 512, 4);
            const uint64_t adl = tc::sdesc(al + arow * 64, 64, 512, 4);
            // B = [dz2 hi | dz2 lo] as ONE N = 128 MN-major operand: the two 64-wide N blocks are the
            // hi and lo tiles, BW_B_BYTES apart (LBO)
            const uint64_t bdh = tc::sdesc(bh + ks * 16 * 128, BW_B_BYTES, 1024, 2);
            tc::mma2_f16(dm, dx, adh, adl, bdh, BW_IDESC2, BW_IDESC, !first || ks != 0);
          }
          if (last) tc::mma_commit(&tfull[ky]);
          if (ky == 2) tc::mma_commit(&empty[stage]);
        }
        __syncwarp();
      }
      if (++stage == BW_STAGES) { stage = 0; phase ^= 1; }
    }
  } else {
    const int ew = warp & 3;                 // TMEM lane quarter
    const int hc = (warp - 2) >> 2;          // column group (o 16 hc .. 16 hc + 15)
    const int row = ew * 32 + lane;          // M row = kx * 32 + ci (quarter 3: kx = 3, unused rows)
    float run[3][BW_EPI_COLS];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < BW_EPI_COLS; ++j) run[i][j] = 0.f;
    for (int blk = 1; blk < nblocks; blk += 2) {  // one drain per pair of blocks
      const int n = c * B + b0 + blk / BW_NKB;
      const float inv = 1.f / (a1scale[n] * dzscale[n]);  // exact: powers of two
#pragma unroll
      for (int ky = 0; ky < 3; ++ky) {
        tc::mbar_wait(&tfull[ky], (blk >> 1) & 1);
        tc::tc_fence_after();
        if (ew == 3) {  // the kx = 3 rows carry no weight: nothing to drain
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&tempty[ky]);
          continue;
        }
        uint32_t vm[BW_EPI_COLS], vx[BW_EPI_COLS];
        const uint32_t base = tmem + ((uint32_t)(ew * 32) << 16) + ky * 2 * C2 + hc * BW_EPI_COLS;
        tc::tmem_ld16(base, vm);
        tc::tmem_ld16(base + C2, vx);
        tc::tmem_ld_wait();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&tempty[ky]);
#pragma unroll
        for (int j = 0; j < BW_EPI_COLS; ++j) run[ky][j] += (__uint_as_float(vm[j]) + __uint_as_float(vx[j])) * inv;
      }
    }
    const int kx = row >> 5, ci = row & 31;
    float* dc = delta + (int64_t)c * ld;
    if (split > 1) {  // partial [ky][o][kx * 32 + ci] of this sample range
      float* wp = wpart + (int64_t)blockIdx.x * BW_PART;
      if (kx < 3)
#pragma unroll
        for (int ky = 0; ky < 3; ++ky)
#pragma unroll
          for (int j = 0; j < BW_EPI_COLS; ++j) wp[(ky * C2 + hc * BW_EPI_COLS + j) * 96 + row] = run[ky][j];
    } else if (kx < 3) {
#pragma unroll
      for (int ky = 0; ky < 3; ++ky)
#pragma unroll
        for (int j = 0; j < BW_EPI_COLS; ++j) {
          const int o = hc * BW_EPI_COLS + j;
          float& dl = dc[O_W2 + (int64_t)o * (C1 * 9) + ci * 9 + ky * 3 + kx];
          dl += st.lr * (run[ky][j] - st.mu * dl);
        }
    }
    const int e = threadIdx.x - 64;
    if (split == 1 && e < C2) {  // conv2 bias: sum of the client's per-sample partials
      const int nb = nbc;
      float gb = 0.f;
      for (int b = 0; b < nb; ++b) gb += db2[(int64_t)(c * B + b) * C2 + e];
      float& dl = dc[O_B2 + e];
      dl += st.lr * (gb - st.mu * dl);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc<512>(tmem);
}

// split conv2 weight gradient: sum the CTA partials of each client in fixed order and
// apply delta += lr * (g - mu * delta) (conv2 weights and bias)
__global__ void conv2_bwd_w_reduce_kernel(const float* __restrict__ wpart, int split, int B,
                                          const int32_t* __restrict__ client_nb, const float* __restrict__ db2,
                                          float* __restrict__ delta, int64_t ld, Step st) {
  const int c = blockIdx.x;
  const int nb = client_nb[c];
  if (nb == 0) return;
  float* dc = delta + (int64_t)c * ld;
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < BW_PART; e += gridDim.y * blockDim.x) {
    float g = 0.f;
    for (int p = 0; p < split; ++p)  // (a part with an empty sample range wrote nothing)
      if ((p + 1) * nb / split > p * nb / split) g += wpart[((int64_t)c * split + p) * BW_PART + e];
    const int row = e % 96, ko = e / 96, o = ko % C2, ky = ko / C2, kx = row >> 5, ci = row & 31;
    float& dl = dc[O_W2 + (int64_t)o * (C1 * 9) + ci * 9 + ky * 3 + kx];
    dl += st.lr * (g - st.mu * dl);
  }
  if (blockIdx.y == 0 && threadIdx.x < C2) {
    float gb = 0.f;
    for (int b = 0; b < nb; ++b) gb += db2[(int64_t)(c * B + b) * C2 + threadIdx.x];
    float& dl = dc[O_B2 + threadIdx.x];
    dl += st.lr * (gb - st.mu * dl);
  }
}

// ------------------------------------------------------------- workspace
struct Work {
  int64_t* slot_row;
  int32_t* slot_client;
  int32_t* client_nb;
  int64_t* prefix;
  double* slot_loss;
  int32_t* slot_hit;
  float *a1, *pooled, *part, *dz3, *dp, *dz1, *db2, *a1scale, *dzscale, *wscale;
  float *gram, *acoef;  // factored fc1 (pooled / dz3 / client_nb then hold hist_steps steps)
  double* gram_part;    // [Cmax][GR_KS][GMAX][FC_RMAX] split-K Gram partials
  __half *pfh, *pfl, *dz3fh, *dz3fl, *thTh, *thTl, *thh, *thl;  // tcgen05 fc1 operands
  float *pscale, *dz3scale, *tscale;
  unsigned* tmax;
  unsigned* umax;     // factored fc1 aggregate: cohort max |U'|
  __half* uprime;     // [Cmax][hi|lo][FC_RMAX][HID]
  float* aggpart;     // [FAG_CHUNKS][FLAT][HID]
  __half *a1fh, *a1fl, *dzfh, *dzfl;
  uint8_t* code;
  uint8_t* wimg;  // per-group conv2 weight images (tcgen05 B operand)
};

inline int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

// layout for N slots and up to Cmax clients
inline int64_t carve(void* base, int N, int Cmax, int H, Work* w) {
  const int64_t hs = H > 1 ? H : 1;
  int64_t off = 0;
  auto take = [&](int64_t bytes) {
    const int64_t o = off;
    off += align256(bytes);
    return o;
  };
  const int64_t o_row = take(8LL * N), o_cl = take(4LL * N), o_nb = take(4LL * hs * (Cmax + 1)),
                o_pre = take(8LL * (Cmax + 1)), o_loss = take(8LL * N), o_hit = take(4LL * N),
                o_a1 = take(4LL * N * A1), o_pool = take(4LL * hs * N * FLAT), o_code = take((int64_t)N * FLAT),
                o_part = take(4LL * KSPLIT * N * HID), o_dz3 = take(4LL * hs * N * HID), o_dp = take(4LL * N * FLAT),
                o_dz1 = take(4LL * N * A1), o_wimg = take((int64_t)WIMG_BYTES * (Cmax + 1)),
                o_db2 = take(4LL * N * C2), o_a1fh = take(2LL * N * A1), o_a1fl = take(2LL * N * A1),
                o_dzfh = take(2LL * N * S2 * S2 * C2), o_dzfl = take(2LL * N * S2 * S2 * C2),
                o_a1s = take(4LL * N), o_dzs = take(4LL * N), o_ws = take(4LL * (Cmax + 1)),
                o_gram = H > 0 ? take(4LL * Cmax * FC_RMAX * FC_RMAX) : 0,
                o_gpart = H > 0 ? take(8LL * Cmax * GR_KS * GMAX * FC_RMAX) : 0,
                o_acoef = H > 0 ? take(4LL * Cmax * GMAX * FC_RMAX) : 0,
                o_pfh = take(2LL * hs * N * FLAT), o_pfl = take(2LL * hs * N * FLAT), o_dz3fh = take(2LL * N * HID),
                o_dz3fl = take(2LL * N * HID), o_thTh = take(2LL * FLAT * HID), o_thTl = take(2LL * FLAT * HID),
                o_thh = take(2LL * FLAT * HID), o_thl = take(2LL * FLAT * HID), o_psc = take(4LL * hs * N),
                o_dz3sc = take(4LL * N), o_tsc = take(16),
                o_u = H > 0 ? take(2LL * Cmax * 2 * FC_RMAX * HID) : 0,          // factored aggregate: U' hi / lo
                o_agp = H > 0 ? take(4LL * FAG_CHUNKS * FLAT * HID) : 0;         // its per-chunk partials
  if (w && base) {
    char* b = static_cast<char*>(base);
    w->slot_row = reinterpret_cast<int64_t*>(b + o_row);
    w->slot_client = reinterpret_cast<int32_t*>(b + o_cl);
    w->client_nb = reinterpret_cast<int32_t*>(b + o_nb);
    w->prefix = reinterpret_cast<int64_t*>(b + o_pre);
    w->slot_loss = reinterpret_cast<double*>(b + o_loss);
    w->slot_hit = reinterpret_cast<int32_t*>(b + o_hit);
    w->a1 = reinterpret_cast<float*>(b + o_a1);
    w->wimg = reinterpret_cast<uint8_t*>(b + o_wimg);
    w->db2 = reinterpret_cast<float*>(b + o_db2);
    w->a1fh = reinterpret_cast<__half*>(b + o_a1fh);
    w->a1fl = reinterpret_cast<__half*>(b + o_a1fl);
    w->dzfh = reinterpret_cast<__half*>(b + o_dzfh);
    w->dzfl = reinterpret_cast<__half*>(b + o_dzfl);
    w->a1scale = reinterpret_cast<float*>(b + o_a1s);
    w->dzscale = reinterpret_cast<float*>(b + o_dzs);
    w->wscale = reinterpret_cast<float*>(b + o_ws);
    w->gram = H > 0 ? reinterpret_cast<float*>(b + o_gram) : nullptr;
    w->gram_part = H > 0 ? reinterpret_cast<double*>(b + o_gpart) : nullptr;
    w->acoef = H > 0 ? reinterpret_cast<float*>(b + o_acoef) : nullptr;
    w->pfh = reinterpret_cast<__half*>(b + o_pfh);
    w->pfl = reinterpret_cast<__half*>(b + o_pfl);
    w->dz3fh = reinterpret_cast<__half*>(b + o_dz3fh);
    w->dz3fl = reinterpret_cast<__half*>(b + o_dz3fl);
    w->thTh = reinterpret_cast<__half*>(b + o_thTh);
    w->thTl = reinterpret_cast<__half*>(b + o_thTl);
    w->thh = reinterpret_cast<__half*>(b + o_thh);
    w->thl = reinterpret_cast<__half*>(b + o_thl);
    w->pscale = reinterpret_cast<float*>(b + o_psc);
    w->dz3scale = reinterpret_cast<float*>(b + o_dz3sc);
    w->tscale = reinterpret_cast<float*>(b + o_tsc);
    w->tmax = reinterpret_cast<unsigned*>(b + o_tsc + 4);
    w->umax = reinterpret_cast<unsigned*>(b + o_tsc + 8);
    w->uprime = H > 0 ? reinterpret_cast<__half*>(b + o_u) : nullptr;
    w->aggpart = H > 0 ? reinterpret_cast<float*>(b + o_agp) : nullptr;
    w->pooled = reinterpret_cast<float*>(b + o_pool);
    w->code = reinterpret_cast<uint8_t*>(b + o_code);
    w->part = reinterpret_cast<float*>(b + o_part);
    w->dz3 = reinterpret_cast<float*>(b + o_dz3);
    w->dp = reinterpret_cast<float*>(b + o_dp);
    w->dz1 = reinterpret_cast<float*>(b + o_dz1);
  }
  return off;
}

int g_num_sms = 148;

int set_smem_limits() {
  static bool done = false;
  if (done) return FB_OK;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(conv2_fwd_pool_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, C2F_SMEM);
  cudaFuncSetAttribute(conv2_bwd_x_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, C2X_SMEM);
  cudaFuncSetAttribute(conv2_bwd_w_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, C2W_SMEM);
  cudaFuncSetAttribute(conv2_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FW_SMEM);
  cudaFuncSetAttribute(conv2_fwd_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FW2_SMEM);
  cudaFuncSetAttribute(fc1_agg_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FAG_SMEM);
  cudaFuncSetAttribute(conv2_bwd_x_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, BX_SMEM);
  cudaFuncSetAttribute(dz2_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, DZB_SMEM);
  cudaFuncSetAttribute(fc1_bwd_fact_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, FC1F_SMEM);
  cudaFuncSetAttribute(fc1_bwd_fact_kernel<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, FC1F_SMEM);
  cudaFuncSetAttribute(fc1_bwd_fact_kernel<GMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, FC1F_SMEM);
  cudaFuncSetAttribute(fc1_materialize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FC1M_SMEM);
  cudaFuncSetAttribute(fc1_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FT_SMEM);
  cudaFuncSetAttribute(conv2_bwd_w_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, BW_SMEM);
  cudaFuncSetAttribute(conv1_bwd_w_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, W1_SMEM);
  cudaFuncSetAttribute(conv1_bwd_w_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, W1_SMEM);
  cudaFuncSetAttribute(conv1_bwd_w_ffma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, WF_SMEM);
  cudaFuncSetAttribute(conv1_bwd_w_ffma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, WF_SMEM);
  cudaFuncSetAttribute(conv1_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, C1F_SMEM);
  cudaFuncSetAttribute(conv1_fwd_ig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, CIG_SMEM);
  cudaFuncSetAttribute(fc1_mat_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FMT_SMEM);
  cudaFuncSetAttribute(conv2_wimg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, WIMG_BYTES);
  cudaFuncSetAttribute(conv2_wimgT_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, WIMGT_BYTES);
  done = true;
  return launch_status("cnn: cudaFuncSetAttribute");
}

// fc1 at theta_t on tcgen05: evaluation and factored training with the tcgen05 conv path
inline bool fc1_tc(const float* delta, bool shared_fc1) { return g_conv_impl == 1 && (!delta || shared_fc1); }

// CTAs per client for the per-client kernels when a launch has few clients (a
// rank's shard at N > 1): split each client's B slots into d groups (d | B)
// until the grid fills one wave of `per_sm` CTAs per SM.
inline int client_split(int clients, int B, int per_sm) {
  int d = 1;
  while (clients * d < g_num_sms * per_sm) {
    int nd = d + 1;
    while (nd <= B && B % nd) ++nd;
    if (nd > B) break;
    d = nd;
  }
  return d;
}

// fp16 images of theta_t's fc1 weights for the tcgen05 fc1 kernels
int prep_theta_images(const float* theta, const Work& w, cudaStream_t s) {
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  cudaMemsetAsync(w.tmax, 0, sizeof(unsigned), s);
  FB_LAUNCH("fc1_theta_max_kernel", s, fc1_theta_max_kernel<<<296, 256, 0, s>>>(theta, w.tmax));
  FB_LAUNCH("fc1_theta_img_kernel", s, fc1_theta_img_kernel<<<FLAT / 64, 256, 0, s>>>(theta, w.tmax, w.thTh, w.thTl,
                                                                                      w.thh, w.thl, w.tscale));
  return launch_status("cnn fc1 theta images");
}

// forward of N slots (shared weights when delta == nullptr) up to the head
// `active`: clients with a slot this step (host-known; sizes the per-client CTA split), -1 = all
int forward(const float* X, const float* theta, const float* delta, int64_t ld, int B, int N, int G,
            const Work& w, cudaStream_t s, const int32_t* client_nb, bool shared_fc1 = false, int active = -1) {
  if (active < 0) active = N / B;
  const bool tc = g_conv_impl == 1;
  if (tc) {
    // slots per CTA: (part of) one client's batch (its own weights), or 16 at theta_t
    const int g1 = delta ? B / client_split(active, B, 2) : C1F_GMAX;
    if (g_conv1_fwd_impl == 1)
      FB_LAUNCH("conv1_fwd_ig_kernel", s, conv1_fwd_ig_kernel<<<(N + g1 - 1) / g1, C1F_THREADS, CIG_SMEM, s>>>(
                                              X, w.slot_row, theta, delta, ld, B, N, g1, w.a1fh, w.a1fl, w.a1scale));
    else
      FB_LAUNCH("conv1_fwd_tc_kernel", s, conv1_fwd_tc_kernel<<<(N + g1 - 1) / g1, C1F_THREADS, C1F_SMEM, s>>>(
                                              X, w.slot_row, theta, delta, ld, B, N, g1, w.a1fh, w.a1fl, w.a1scale));
  } else {
    FB_LAUNCH("conv1_fwd_kernel", s, conv1_fwd_kernel<<<N, 256, 0, s>>>(X, w.slot_row, theta, delta, ld, B, w.a1,
                                                                        nullptr, nullptr, w.a1scale));
  }
  if (tc) {
    // weight groups: one per client in training (G = B), one shared image at theta_t in evaluation
    const int groups = delta ? (N + B - 1) / B : 1;
    FB_LAUNCH("conv2_wimg_kernel", s, conv2_wimg_kernel<<<groups, 256, WIMG_BYTES, s>>>(theta, delta, ld, client_nb, w.wimg,
                                                                                   w.wscale));
    CUtensorMap mh, ml;
    int st = a1f_tensor_map(&mh, w.a1fh, N, S1, FW_BAND);
    if (!st) st = a1f_tensor_map(&ml, w.a1fl, N, S1, FW_BAND);
    if (st) return st;
#ifndef FW_EVAL_G
#define FW_EVAL_G 8
#endif
    const int gt = delta ? B / client_split(active, B, 1) : FW_EVAL_G;  // samples per CTA
    if (g_conv2_pairs)  // one CTA pair per former CTA's samples (cluster dims 2)
      FB_LAUNCH("conv2_fwd_tc_kernel", s, conv2_fwd_tc2_kernel<<<2 * ((N + gt - 1) / gt), FW_THREADS, FW2_SMEM, s>>>(
            mh, ml, w.wimg, w.wscale, delta ? 0 : 1, w.slot_row, N, gt, theta, delta, ld, B, w.a1scale, w.pooled,
            w.code));
    else
      FB_LAUNCH("conv2_fwd_tc_kernel", s, conv2_fwd_tc_kernel<<<(N + gt - 1) / gt, FW_THREADS, FW_SMEM, s>>>(
            mh, ml, w.wimg, w.wscale, delta ? 0 : 1, w.slot_row, N, gt, theta, delta, ld, B, w.a1scale, w.pooled,
            w.code));
  } else {
    FB_LAUNCH("conv2_fwd_pool_kernel", s, conv2_fwd_pool_kernel<<<N, 256, C2F_SMEM, s>>>(w.a1, nullptr, w.slot_row, theta, delta, ld, B, w.pooled, w.code));
  }
  if (fc1_tc(delta, shared_fc1)) {
    FB_LAUNCH("pooled_split_kernel", s, pooled_split_kernel<<<N, 256, 0, s>>>(w.pooled, w.slot_row, w.pfh, w.pfl,
                                                                               w.pscale));
    CUtensorMap ah, al, bh, bl;
    int st = tensor_map_2d_f16(&ah, w.pfh, FLAT, N, FT_KS, 128);
    if (!st) st = tensor_map_2d_f16(&al, w.pfl, FLAT, N, FT_KS, 128);
    if (!st) st = tensor_map_2d_f16(&bh, w.thTh, FLAT, HID, FT_KS, 128);
    if (!st) st = tensor_map_2d_f16(&bl, w.thTl, FLAT, HID, FT_KS, 128);
    if (st) return st;
    FtArgs fa{0, N, (N + 127) / 128, 0, w.pscale, w.tscale, w.part};
    fa.units = fa.mtiles * FT_FSPLIT;
    FB_LAUNCH("fc1_tc_kernel", s, fc1_tc_kernel<<<std::min(fa.units, g_num_sms), TC_THREADS, FT_SMEM, s>>>(
                                      ah, al, bh, bl, fa));
  } else {
    // weight-sharing group per warp: the client's B slots in training, 8 rows at theta_t in evaluation
    // (factored fc1: every slot at theta_t, the history correction is applied in the head)
    const float* fd = shared_fc1 ? nullptr : delta;
    const int gf = fd ? G : 8;
    const dim3 grid((N + gf - 1) / gf, KSPLIT);
    if (gf <= 8)
      FB_LAUNCH("fc1_fwd_kernel", s, fc1_fwd_kernel<8><<<grid, FF_WARPS * 32, 0, s>>>(w.pooled, w.slot_row, N, gf, theta, fd, ld, w.part));
    else if (gf <= 10)
      FB_LAUNCH("fc1_fwd_kernel", s, fc1_fwd_kernel<10><<<grid, FF_WARPS * 32, 0, s>>>(w.pooled, w.slot_row, N, gf, theta, fd, ld, w.part));
    else if (gf <= 12)
      FB_LAUNCH("fc1_fwd_kernel", s, fc1_fwd_kernel<12><<<grid, FF_WARPS * 32, 0, s>>>(w.pooled, w.slot_row, N, gf, theta, fd, ld, w.part));
    else
      FB_LAUNCH("fc1_fwd_kernel", s, fc1_fwd_kernel<GMAX><<<grid, FF_WARPS * 32, 0, s>>>(w.pooled, w.slot_row, N, gf, theta, fd, ld, w.part));
  }
  return launch_status("cnn forward");
}

}  // namespace cnn
}  // namespace fb

using namespace fb::cnn;

extern "C" {

#ifdef FB_FWD_PROF
int fb_debug_prof(unsigned long long* out) {  // timing experiments only
  cudaMemcpyFromSymbol(out, g_prof, sizeof(unsigned long long) * 8);
  unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyToSymbol(g_prof, z, sizeof(z));
  return 0;
}
#endif

int fb_cnn_fc1_aggregate_f32(const float* coef, int num_clients, int batch_size, int max_steps, float lr,
                             float prox_mu, int max_slots, int hist_steps, void* workspace, int64_t workspace_bytes,
                             float* agg_fc1, void* stream) {
  using namespace fb::cnn;
  FB_REQUIRE(num_clients >= 1 && batch_size >= 1 && batch_size <= GMAX && max_steps >= 1 && hist_steps >= max_steps &&
                 hist_steps * batch_size <= FC_RMAX && max_slots >= batch_size,
             "cnn_fc1_aggregate: bad arguments");
  const int per = max_slots / batch_size;
  FB_REQUIRE(num_clients <= per, "cnn_fc1_aggregate: the cohort must have run as one wave (%d > %d clients)",
             num_clients, per);
  FB_REQUIRE(workspace_bytes >= carve(nullptr, max_slots, per, hist_steps, nullptr),
             "cnn_fc1_aggregate: workspace too small");
  int st = set_smem_limits();
  if (st) return st;
  cudaStream_t s = fb::as_stream(stream);
  Work w;
  FB_REQUIRE(reinterpret_cast<uintptr_t>(workspace) % 256 == 0, "cnn: workspace must be 256-byte aligned");
  carve(workspace, max_slots, per, hist_steps, &w);
  const int B = batch_size, C = num_clients, N = C * B;
  Hist hs{};
  hs.phist = w.pooled;
  hs.pstride = (int64_t)N * FLAT;
  hs.dz3h = w.dz3;
  hs.dstride = (int64_t)N * HID;
  hs.nbh = w.client_nb;
  hs.cstride = per + 1;
  cudaMemsetAsync(w.umax, 0, sizeof(unsigned), s);
  FB_LAUNCH("fc1_umax_kernel", s, fc1_umax_kernel<<<C, 256, 0, s>>>(hs, w.pscale, coef, N, max_steps, B, lr,
                                                                    prox_mu, w.umax));
  FB_LAUNCH("fc1_ubuild_kernel", s, fc1_ubuild_kernel<<<C, 256, 0, s>>>(hs, w.pscale, coef, N, max_steps, B, lr,
                                                                        prox_mu, w.umax, w.uprime));
  CUtensorMap mh, ml, mu;
  st = hist_tensor_map(&mh, w.pfh, N, max_steps, B);
  if (!st) st = hist_tensor_map(&ml, w.pfl, N, max_steps, B);
  if (!st) st = tensor_map_2d_f16(&mu, w.uprime, HID, (int64_t)C * 2 * FC_RMAX, 64, FC_RMAX);
  if (st) return st;
  const int chunk = (C + FAG_CHUNKS - 1) / FAG_CHUNKS;
  FB_LAUNCH("fc1_agg_tc_kernel", s, fc1_agg_tc_kernel<<<dim3(FMT_TILES, FAG_CHUNKS), FMT_THREADS, FAG_SMEM, s>>>(
                                        mh, ml, mu, C, max_steps, B, chunk, w.umax, w.aggpart));
  FB_LAUNCH("fc1_agg_reduce_kernel", s, fc1_agg_reduce_kernel<<<g_num_sms * 4, 256, 0, s>>>(w.aggpart, FAG_CHUNKS,
                                                                                          agg_fc1));
  return fb::launch_status("cnn_fc1_aggregate");
}

int fb_cnn_set_conv_impl(int impl) {
  FB_REQUIRE(impl >= 0 && impl <= 4,
             "fb_cnn_set_conv_impl: 0 (FP32 CUDA cores), 1 (tcgen05), 2 (tcgen05, CTA-pair conv2 forward), 3 "
             "(tcgen05, im2col-staged conv1 forward) or 4 (tcgen05, FP32 conv1 weight gradient)");
  fb::cnn::g_conv_impl = impl == 0 ? 0 : 1;
  fb::cnn::g_conv2_pairs = impl == 2;
  fb::cnn::g_conv1_fwd_impl = impl == 3 ? 0 : 1;
  fb::cnn::g_conv1_bwd_ffma = impl == 4;
  return FB_OK;
}

int64_t fb_cnn_workspace_bytes(int max_slots, int max_clients, int hist_steps) {
  if (max_slots < 0 || max_clients < 0 || hist_steps < 0) return -1;
  return carve(nullptr, max_slots, max_clients, hist_steps, nullptr);
}

int fb_eval_cnn_f32(const float* theta, const float* X, const int32_t* y, const int64_t* row_start,
                    const int32_t* num_rows, int num_clients, int64_t total_rows, double* loss_sum,
                    int32_t* correct, int max_slots, void* workspace, int64_t workspace_bytes,
                    const int32_t* perms, const int64_t* perm_off, int skip, void* stream) {
  FB_REQUIRE(num_clients >= 0 && total_rows >= 0 && max_slots >= GMAX, "eval_cnn: bad arguments");
  FB_REQUIRE(workspace_bytes >= carve(nullptr, max_slots, num_clients, 0, nullptr), "eval_cnn: workspace too small");
  if (num_clients == 0) return FB_OK;
  int st = set_smem_limits();
  if (st) return st;
  cudaStream_t s = fb::as_stream(stream);
  Work w;
  FB_REQUIRE(reinterpret_cast<uintptr_t>(workspace) % 256 == 0, "cnn: workspace must be 256-byte aligned");
  carve(workspace, max_slots, num_clients, 0, &w);
  const int N = (max_slots / GMAX) * GMAX;
  cudaMemsetAsync(loss_sum, 0, sizeof(double) * num_clients, s);
  cudaMemsetAsync(correct, 0, sizeof(int32_t) * num_clients, s);
  FB_REQUIRE(!perms || (perm_off && skip >= 0), "eval_cnn: perms need perm_off and skip >= 0");
  FB_LAUNCH("prefix_kernel", s, prefix_kernel<<<1, 1, 0, s>>>(num_rows, num_clients, w.prefix, perms ? skip : 0));
  const bool tcf = fc1_tc(nullptr, false);
  if (tcf) {
    st = prep_theta_images(theta, w, s);
    if (st) return st;
  }
  for (int64_t r0 = 0; r0 < total_rows; r0 += N) {
    FB_LAUNCH("eval_slots_kernel", s, eval_slots_kernel<<<(N + 255) / 256, 256, 0, s>>>(r0, N, total_rows, w.prefix, num_clients, row_start,
                                                      w.slot_row, w.slot_client, perms, perm_off, num_rows, skip));
    st = forward(X, theta, nullptr, 0, 1, N, GMAX, w, s, nullptr);
    if (st) return st;
    FB_LAUNCH("head_kernel", s, head_kernel<<<N / GMAX, HID, 0, s>>>(w.part, w.slot_row, N, GMAX, y, theta, nullptr, 0, nullptr, Step{0, 0},
                                         nullptr, w.slot_loss, w.slot_hit, Hist{}, tcf ? FT_FSPLIT : KSPLIT,
                                         nullptr, nullptr, nullptr));
    FB_LAUNCH("eval_reduce_kernel", s, eval_reduce_kernel<<<(num_clients + 127) / 128, 128, 0, s>>>(w.slot_loss, w.slot_hit, w.slot_client, N, r0,
                                                                 w.prefix, num_clients, loss_sum, correct));
    st = fb::launch_status("eval_cnn");
    if (st) return st;
  }
  return FB_OK;
}

// SCAFFOLD control term of one local step (fedsim/models/kernels.py:66-67,117-120 with
// c = c - c_i, fedsim/algorithms/scaffold.py:46-57): delta_c += lr * corr_c for every
// client that took this step (nb > 0); float4 over the row, tail past D masked
__global__ void control_step_kernel(float* __restrict__ delta, int64_t ld, const float* __restrict__ corr,
                                    int64_t ldc, int C, const int32_t* __restrict__ nb, float lr) {
  const int64_t q = (D + 3) / 4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)C * q;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / q);
    const int64_t j = i - (int64_t)c * q;
    if (nb[c] == 0) continue;
    float4 d = reinterpret_cast<float4*>(delta + (int64_t)c * ld)[j];
    const float4 g = __ldg(reinterpret_cast<const float4*>(corr + (int64_t)c * ldc) + j);
    const int64_t e = 4 * j;
    d.x = fmaf(lr, g.x, d.x);
    if (e + 1 < D) d.y = fmaf(lr, g.y, d.y);
    if (e + 2 < D) d.z = fmaf(lr, g.z, d.z);
    if (e + 3 < D) d.w = fmaf(lr, g.w, d.w);
    reinterpret_cast<float4*>(delta + (int64_t)c * ld)[j] = d;
  }
}

int fb_local_sgd_cnn_f32(const float* theta_t, const float* X, const int32_t* y, const int64_t* row_start,
                         const int32_t* num_rows, const int32_t* perms, const int64_t* perm_off, int num_clients,
                         int epochs, int batch_size, int max_steps, float lr, float prox_mu, float* delta_out,
                         int64_t ld_delta, int32_t* nonfinite, int max_slots, int hist_steps, void* workspace,
                         int64_t workspace_bytes, double* fc1_sumsq, const float* control, int64_t ld_control,
                         const int32_t* h_client_steps, int fc1_store, double* eval_loss, int32_t* eval_correct,
                         void* stream) {
  FB_REQUIRE(num_clients >= 0 && epochs >= 0 && batch_size >= 1 && max_steps >= 0 && hist_steps >= 0,
             "local_sgd_cnn: bad arguments");
  FB_REQUIRE(fc1_store || (hist_steps > 0 && fc1_sumsq && g_conv_impl == 1 && num_clients <= max_slots / batch_size),
             "local_sgd_cnn: fc1_store = 0 needs the factored tcgen05 form, fc1_sumsq and one wave of clients");
  FB_REQUIRE(!control || (hist_steps == 0 && ld_control >= D && (ld_control & 3) == 0),
             "local_sgd_cnn: control variates need the dense fc1 form (hist_steps 0) and ld_control >= D, "
             "a multiple of 4");
  FB_UNSUPPORTED(batch_size <= GMAX, "local_sgd_cnn: batch_size %d > %d", batch_size, GMAX);
  FB_REQUIRE(ld_delta >= D && (ld_delta & 3) == 0, "local_sgd_cnn: ld_delta must be >= D and a multiple of 4");
  FB_REQUIRE(max_slots >= batch_size, "local_sgd_cnn: max_slots < batch_size");
  FB_REQUIRE(hist_steps == 0 || (hist_steps >= max_steps && hist_steps * batch_size <= FC_RMAX),
             "local_sgd_cnn: hist_steps must be 0 (dense fc1) or >= max_steps with hist_steps*batch_size <= %d",
             FC_RMAX);
  const int per = max_slots / batch_size;  // clients per wave
  FB_REQUIRE(workspace_bytes >= carve(nullptr, max_slots, per, hist_steps, nullptr),
             "local_sgd_cnn: workspace too small");
  if (num_clients == 0) return FB_OK;
  int st = set_smem_limits();
  if (st) return st;
  cudaStream_t s = fb::as_stream(stream);
  Work w;
  FB_REQUIRE(reinterpret_cast<uintptr_t>(workspace) % 256 == 0, "cnn: workspace must be 256-byte aligned");
  carve(workspace, max_slots, per, hist_steps, &w);
  const bool fact = hist_steps > 0;
  const int64_t tot4 = (int64_t)num_clients * (ld_delta / 4);
  // factored fc1: the fc1 weight block is written whole by fc1_materialize
  FB_LAUNCH("zero_delta_kernel", s, zero_delta_kernel<<<(unsigned)std::min<int64_t>((tot4 + 255) / 256, 148 * 16), 256, 0, s>>>(
                                        delta_out, ld_delta, num_clients, fact ? O_F1 : 0, fact ? O_BF1 : 0));
  cudaMemsetAsync(nonfinite, 0, sizeof(int32_t) * num_clients, s);
  const Step sp{lr, prox_mu};
  const int B = batch_size;
  const bool tcf = fc1_tc(delta_out, fact);
  if (tcf) {
    st = prep_theta_images(theta_t, w, s);
    if (st) return st;
  }
  for (int c0 = 0; c0 < num_clients; c0 += per) {
    const int Cw = min(per, num_clients - c0);
    const int N = Cw * B;
    float* dlt = delta_out + (int64_t)c0 * ld_delta;
    Hist hs{};
    if (fact) {
      hs.phist = w.pooled;
      hs.pstride = (int64_t)N * FLAT;
      hs.dz3h = w.dz3;
      hs.dstride = (int64_t)N * HID;
      hs.nbh = w.client_nb;
      hs.cstride = per + 1;
      hs.gram = w.gram;
      hs.R = FC_RMAX;
      hs.acoef = w.acoef;
    }
    for (int step = 0; step < max_steps; ++step) {
      Work ws = w;  // this step's slices of the history buffers
      if (fact) {
        ws.pooled = w.pooled + step * hs.pstride;
        ws.pfh = w.pfh + step * hs.pstride;  // fp16 hi / lo pooled history (tcgen05 fc1 materialize)
        ws.pfl = w.pfl + step * hs.pstride;
        ws.pscale = w.pscale + (int64_t)step * N;
        ws.dz3 = w.dz3 + step * hs.dstride;
        ws.client_nb = w.client_nb + step * hs.cstride;
        hs.s = step;
      }
      FB_LAUNCH("train_slots_kernel", s, train_slots_kernel<<<(N + 255) / 256, 256, 0, s>>>(step, row_start + c0, num_rows + c0, perms, perm_off + c0,
                                                        Cw, epochs, B, ws.slot_row, ws.client_nb));
      int active = Cw;  // clients still training at this step (ragged cohorts: a few long clients)
      if (h_client_steps) {
        active = 0;
        for (int c = 0; c < Cw; ++c) active += h_client_steps[c0 + c] > step;
        active = std::max(active, 1);
      }
      st = forward(X, theta_t, dlt, ld_delta, B, N, B, ws, s, ws.client_nb, fact, active);
      const int rs = active * KSPLIT < 4 * g_num_sms ? 7 : 1;
      if (st) return st;
      if (fact) {
        FB_REQUIRE((int64_t)max_steps * N * FLAT < (1LL << 31), "local_sgd_cnn: factored-fc1 history exceeds 2^31 elements");
#ifndef GR_NKS
#define GR_NKS 7
#endif
        const int gks = Cw * GR_NKS >= 4 * g_num_sms ? GR_NKS : 14;  // more K splits for a small shard
        FB_REQUIRE(Cw <= 65535, "local_sgd_cnn: %d clients in one wave exceed the Gram grid's z extent", Cw);
        const dim3 ggrid(std::min(GR_Z, (int)((step + 1) * B + GR_JW * GR_WARPS - 1) / (GR_JW * GR_WARPS)), gks, Cw);
        if (B <= 8)
          FB_LAUNCH("fc1_gram_split_kernel", s, fc1_gram_split_kernel<8><<<ggrid, GR_WARPS * 32, 0, s>>>(
                                                    hs, B, w.gram_part));
        else if (B <= 10)
          FB_LAUNCH("fc1_gram_split_kernel", s, fc1_gram_split_kernel<10><<<ggrid, GR_WARPS * 32, 0, s>>>(
                                                    hs, B, w.gram_part));
        else
          FB_LAUNCH("fc1_gram_split_kernel", s, fc1_gram_split_kernel<GMAX><<<ggrid, GR_WARPS * 32, 0, s>>>(
                                                    hs, B, w.gram_part));
        FB_LAUNCH("fc1_gram_reduce_kernel", s, fc1_gram_reduce_kernel<<<Cw, 256, 0, s>>>(hs, B, gks, w.gram_part));
      }
      // step 0 runs at theta_t: its batch's loss / hits are those rows' evaluation (the caller
      // evaluated only the rest, fb_eval_cnn_f32 with skip = batch_size)
      const bool ev0 = step == 0 && eval_loss != nullptr;
      FB_LAUNCH("head_kernel", s, head_kernel<<<Cw, HID, 0, s>>>(ws.part, ws.slot_row, N, B, y, theta_t, dlt, ld_delta, ws.client_nb, sp, ws.dz3,
                                     ev0 ? ws.slot_loss : nullptr, ev0 ? ws.slot_hit : nullptr, hs,
                                     tcf ? FT_FSPLIT : KSPLIT, tcf ? ws.dz3fh : nullptr, ws.dz3fl, ws.dz3scale));
      if (ev0)
        FB_LAUNCH("step0_eval_kernel", s, step0_eval_kernel<<<(Cw + 127) / 128, 128, 0, s>>>(
                                              ws.slot_loss, ws.slot_hit, ws.client_nb, B, Cw, eval_loss + c0,
                                              eval_correct + c0));
      if (tcf) {
        CUtensorMap ah, al, bh, bl;
        st = tensor_map_2d_f16(&ah, ws.dz3fh, HID, N, FT_KS, 128);
        if (!st) st = tensor_map_2d_f16(&al, ws.dz3fl, HID, N, FT_KS, 128);
        if (!st) st = tensor_map_2d_f16(&bh, ws.thh, HID, FLAT, FT_KS, 128);
        if (!st) st = tensor_map_2d_f16(&bl, ws.thl, HID, FLAT, FT_KS, 128);
        if (st) return st;
        FtArgs fa{1, N, (N + 127) / 128, 0, ws.dz3scale, ws.tscale, ws.dp};
        fa.units = fa.mtiles * (FLAT / 128);
        FB_LAUNCH("fc1_tc_kernel", s, fc1_tc_kernel<<<std::min(fa.units, g_num_sms), TC_THREADS, FT_SMEM, s>>>(
                                          ah, al, bh, bl, fa));
        if (step > 0) {
          if (B <= 8)
            FB_LAUNCH("fc1_dp_hist_kernel", s, fc1_dp_hist_kernel<8><<<dim3(Cw, KSPLIT), KCHUNK / 4, 0, s>>>(
                                                  B, ws.client_nb, hs, ws.dp));
          else if (B <= 10)
            FB_LAUNCH("fc1_dp_hist_kernel", s, fc1_dp_hist_kernel<10><<<dim3(Cw, KSPLIT), KCHUNK / 4, 0, s>>>(
                                                  B, ws.client_nb, hs, ws.dp));
          else
            FB_LAUNCH("fc1_dp_hist_kernel", s, fc1_dp_hist_kernel<GMAX><<<dim3(Cw, KSPLIT), KCHUNK / 4, 0, s>>>(
                                                  B, ws.client_nb, hs, ws.dp));
        }
      } else if (fact) {
        if (B <= 8)
          FB_LAUNCH("fc1_bwd_fact_kernel", s, fc1_bwd_fact_kernel<8><<<dim3(Cw, KSPLIT), FB_WARPS * 32, FC1F_SMEM, s>>>(
              ws.dz3, B, ws.client_nb, theta_t, hs, ws.dp));
        else if (B <= 10)
          FB_LAUNCH("fc1_bwd_fact_kernel", s, fc1_bwd_fact_kernel<10><<<dim3(Cw, KSPLIT), FB_WARPS * 32, FC1F_SMEM, s>>>(
              ws.dz3, B, ws.client_nb, theta_t, hs, ws.dp));
        else
          FB_LAUNCH("fc1_bwd_fact_kernel", s, fc1_bwd_fact_kernel<GMAX><<<dim3(Cw, KSPLIT), FB_WARPS * 32, FC1F_SMEM, s>>>(
              ws.dz3, B, ws.client_nb, theta_t, hs, ws.dp));
      } else if (B <= 8) {  // (rs: row split of the dense fc1 update when few clients are active)
        FB_LAUNCH("fc1_bwd_kernel", s, fc1_bwd_kernel<8><<<dim3(Cw, KSPLIT * rs), FB_WARPS * 32, FC1B_SMEM, s>>>(
            ws.pooled, ws.dz3, B, ws.client_nb, theta_t, dlt, ld_delta, sp, ws.dp, rs));
      } else if (B <= 10) {
        FB_LAUNCH("fc1_bwd_kernel", s, fc1_bwd_kernel<10><<<dim3(Cw, KSPLIT * rs), FB_WARPS * 32, FC1B_SMEM, s>>>(
            ws.pooled, ws.dz3, B, ws.client_nb, theta_t, dlt, ld_delta, sp, ws.dp, rs));
      } else {
        FB_LAUNCH("fc1_bwd_kernel", s, fc1_bwd_kernel<GMAX><<<dim3(Cw, KSPLIT * rs), FB_WARPS * 32, FC1B_SMEM, s>>>(
            ws.pooled, ws.dz3, B, ws.client_nb, theta_t, dlt, ld_delta, sp, ws.dp, rs));
      }
      if (g_conv_impl == 1) {
        FB_LAUNCH("dz2_build_kernel", s, dz2_build_kernel<<<N, DZB_THREADS, DZB_SMEM, s>>>(ws.dp, ws.pooled, ws.code, ws.slot_row, ws.dzfh, ws.dzfl, ws.dzscale, ws.db2));
        FB_LAUNCH("conv2_wimgT_kernel", s, conv2_wimgT_kernel<<<Cw, 256, WIMGT_BYTES, s>>>(theta_t, dlt, ld_delta, ws.client_nb,
                                                                                 ws.wimg, ws.wscale));
        CUtensorMap mh, ml;
        st = dzf_tensor_map(&mh, ws.dzfh, N, S1, BX_BAND);
        if (!st) st = dzf_tensor_map(&ml, ws.dzfl, N, S1, BX_BAND);
        if (st) return st;
        const int split = client_split(active, B, 1);
        FB_LAUNCH("conv2_bwd_x_tc_kernel", s, conv2_bwd_x_tc_kernel<<<Cw * split, BX_THREADS, BX_SMEM, s>>>(
            mh, ml, ws.wimg, ws.wscale, ws.slot_row, B / split, B, ws.dzscale, ws.a1fh, ws.a1fl, ws.dz1));
        CUtensorMap ah, al, dh, dl;
        st = a1f_tensor_map(&ah, ws.a1fh, N, S1, BW_ROWS + 2);
        if (!st) st = a1f_tensor_map(&al, ws.a1fl, N, S1, BW_ROWS + 2);
        if (!st) st = dzf_tensor_map(&dh, ws.dzfh, N, S1, BW_ROWS);
        if (!st) st = dzf_tensor_map(&dl, ws.dzfl, N, S1, BW_ROWS);
        if (st) return st;
        // few active clients: split each client's samples over CTAs, partials in the (consumed) dp buffer
        int wsplit = 1;
        while (wsplit < B && active * (wsplit + 1) <= g_num_sms &&
               (int64_t)Cw * (wsplit + 1) * BW_PART <= (int64_t)N * FLAT)
          ++wsplit;
        FB_LAUNCH("conv2_bwd_w_tc_kernel", s, conv2_bwd_w_tc_kernel<<<Cw * wsplit, BW_THREADS, BW_SMEM, s>>>(
            ah, al, dh, dl, B, ws.client_nb, ws.a1scale, ws.dzscale, ws.db2, dlt, ld_delta, sp, wsplit, ws.dp));
        if (wsplit > 1)
          FB_LAUNCH("conv2_bwd_w_reduce_kernel", s, conv2_bwd_w_reduce_kernel<<<dim3(Cw, 8), 256, 0, s>>>(
                                                        ws.dp, wsplit, B, ws.client_nb, ws.db2, dlt, ld_delta, sp));
      } else {
        FB_LAUNCH("conv2_bwd_x_kernel", s, conv2_bwd_x_kernel<<<N, 256, C2X_SMEM, s>>>(ws.dp, ws.pooled, ws.code, ws.a1, ws.slot_row, B, theta_t, dlt,
                                                    ld_delta, ws.dz1));
        FB_LAUNCH("conv2_bwd_w_kernel", s, conv2_bwd_w_kernel<<<Cw, 256, C2W_SMEM, s>>>(ws.dp, ws.pooled, ws.code, ws.a1, nullptr, B, ws.client_nb, dlt, ld_delta,
                                                     sp));
      }
      if (g_conv_impl == 1 && g_conv1_bwd_ffma) {
        int split1 = 1;  // few active clients: split each client's samples over CTAs (1 CTA per SM)
        while (split1 < B && active * (split1 + 1) <= g_num_sms) ++split1;
        if (split1 > 1) {
          FB_LAUNCH("conv1_bwd_w_ffma_kernel", s, conv1_bwd_w_ffma_kernel<true><<<Cw * split1, WF_THREADS, WF_SMEM, s>>>(
                                                      X, ws.slot_row, ws.dz1, B, ws.client_nb, dlt, ld_delta, sp,
                                                      split1, ws.dp));
          FB_LAUNCH("conv1_bwd_w_reduce_kernel", s, conv1_bwd_w_reduce_kernel<<<Cw, 256, 0, s>>>(
                                                        ws.dp, split1, ws.client_nb, dlt, ld_delta, sp));
        } else {
          FB_LAUNCH("conv1_bwd_w_ffma_kernel", s, conv1_bwd_w_ffma_kernel<false><<<Cw, WF_THREADS, WF_SMEM, s>>>(
                                                      X, ws.slot_row, ws.dz1, B, ws.client_nb, dlt, ld_delta, sp,
                                                      1, nullptr));
        }
      } else if (g_conv_impl == 1)
      {
        int split1 = 1;  // few active clients: split each client's samples over CTAs (2 CTAs per SM)
        while (split1 < B && active * (split1 + 1) <= 2 * g_num_sms) ++split1;
        if (split1 > 1) {
          FB_LAUNCH("conv1_bwd_w_tc_kernel", s, conv1_bwd_w_tc_kernel<true><<<Cw * split1, W1_THREADS, W1_SMEM, s>>>(
                                                     X, ws.slot_row, ws.dz1, B, ws.client_nb, dlt, ld_delta, sp,
                                                     split1, ws.dp));
          FB_LAUNCH("conv1_bwd_w_reduce_kernel", s, conv1_bwd_w_reduce_kernel<<<Cw, 256, 0, s>>>(
                                                        ws.dp, split1, ws.client_nb, dlt, ld_delta, sp));
        } else {
          FB_LAUNCH("conv1_bwd_w_tc_kernel", s, conv1_bwd_w_tc_kernel<false><<<Cw, W1_THREADS, W1_SMEM, s>>>(
                                                     X, ws.slot_row, ws.dz1, B, ws.client_nb, dlt, ld_delta, sp,
                                                     1, nullptr));
        }
      }
      else
        FB_LAUNCH("conv1_bwd_w_kernel", s, conv1_bwd_w_kernel<<<Cw, C1B_WARPS * 32, 0, s>>>(
                                                X, ws.slot_row, ws.dz1, B, ws.client_nb, dlt, ld_delta, sp));
      if (control)  // SCAFFOLD: theta -= lr * (g + c - c_i), the gradient part applied above
        FB_LAUNCH("control_step_kernel", s, control_step_kernel<<<g_num_sms * 8, 256, 0, s>>>(
                                                dlt, ld_delta, control + (int64_t)c0 * ld_control, ld_control, Cw,
                                                ws.client_nb, lr));
      st = fb::launch_status("local_sgd_cnn step");
      if (st) return st;
    }
    if (fact && tcf) {
      CUtensorMap mh, ml;
      st = hist_tensor_map(&mh, w.pfh, N, max_steps, B);
      if (!st) st = hist_tensor_map(&ml, w.pfl, N, max_steps, B);
      if (st) return st;
#ifndef FMT_SQ_SPLIT
#define FMT_SQ_SPLIT 1  // squares only: one CTA per client (U' built once; 0.80 vs 1.05 ms at 2)
#endif
      const int fs = fc1_store ? FMT_SPLIT : FMT_SQ_SPLIT;
      const int msplit = Cw * fs >= g_num_sms ? fs : 7;  // CTAs per client (7 for a small shard)
      FB_LAUNCH("fc1_mat_tc_kernel", s, fc1_mat_tc_kernel<<<dim3(Cw, msplit), FMT_THREADS, FMT_SMEM, s>>>(
                                            mh, ml, hs, w.pscale, N, max_steps, B, lr, prox_mu, dlt, ld_delta,
                                            fc1_sumsq ? w.gram_part : nullptr, fc1_store));
      if (fc1_sumsq)
        FB_LAUNCH("fc1_sumsq_reduce_kernel", s, fc1_sumsq_reduce_kernel<<<(Cw + 127) / 128, 128, 0, s>>>(
                                                    w.gram_part, msplit, Cw, w.client_nb, fc1_sumsq + c0));
    } else if (fact) {
      FB_LAUNCH("fc1_materialize_kernel", s, fc1_materialize_kernel<<<dim3(Cw, FLAT / FM_K), 256, FC1M_SMEM, s>>>(
                                                   hs, max_steps, B, lr, prox_mu, dlt, ld_delta));
      if (fc1_sumsq)  // (validation path) the block's squares by a plain pass over it
        FB_LAUNCH("fc1_sumsq_scan_kernel", s, fc1_sumsq_scan_kernel<<<Cw, 256, 0, s>>>(
                                                  dlt, ld_delta, w.client_nb, fc1_sumsq + c0));
    }
  }
  return FB_OK;
}

}  // extern "C"
