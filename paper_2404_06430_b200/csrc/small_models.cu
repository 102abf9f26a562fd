// Batched local SGD and evaluation for the reference-native models:
// multinomial logistic regression (fedsim/models/kernels.py:38-83) and the
// one-hidden-layer ReLU MLP (fedsim/models/kernels.py:86-136).
//
// One CTA owns one client for the whole local fit: the client's current
// parameters, its accumulated delta and the step gradient live in shared
// memory (D = 330 / 2,762 floats at the reference shapes), the minibatch
// rows are gathered from the packed dataset by the client's permutation,
// and every contraction is a few hundred FFMAs per thread -- far below a
// tensor-core tile (K = 32, N = 10), so FP32 FFMA in shared memory is the
// right tool.  The grid is the cohort; at C = 1000 that is ~7 CTAs per SM.
//
// Numerics follow the reference kernels: softmax with the row max
// subtracted, the batch gradient divided by the ACTUAL batch size (the
// tail batch is kept), every parameter updated only after all gradients of
// the step are formed.  The delta theta_t - theta_c is accumulated
// directly (not recovered by a cancelling subtraction at the end).

#include "fb_common.cuh"

namespace fb {
namespace {

constexpr int kThreads = 256;
constexpr int kEvalRows = 32;

struct Dims {
  int d, h, k;  // input dim, hidden units (0 for linear), classes
  __host__ __device__ int D() const { return h ? d * h + h + h * k + k : d * k + k; }
};

// act(r, j): input of the output layer for row r (relu(z1) for the MLP, x for linear)
template <bool kHidden>
__device__ __forceinline__ float act(const float* Xb, const float* Z1, const Dims& m, int r, int j) {
  if constexpr (kHidden) return fmaxf(Z1[r * m.h + j], 0.0f);
  else return Xb[r * m.d + j];
}

template <bool kHidden>
__global__ void __launch_bounds__(kThreads) local_sgd_small_kernel(
    const float* __restrict__ theta_t, Dims m, const float* __restrict__ X,
    const int32_t* __restrict__ y, const int64_t* __restrict__ row_start,
    const int32_t* __restrict__ num_rows, const int32_t* __restrict__ perms,
    const int64_t* __restrict__ perm_off, int epochs, int B, float lr, float mu,
    const float* __restrict__ control, int64_t ld_control, float* __restrict__ delta_out,
    int64_t ld_delta, int32_t* __restrict__ nonfinite) {
  extern __shared__ float smem[];
  const int c = blockIdx.x;
  const int D = m.D();
  const int hin = kHidden ? m.h : m.d;  // width of the output layer's input
  float* W = smem;            // current parameters          [D]
  float* Dl = W + D;          // accumulated delta            [D]
  float* G = Dl + D;          // step gradient                [D]
  float* Xb = G + D;          // batch rows                   [B, d]
  float* Lg = Xb + B * m.d;   // logits -> dloss              [B, k]
  float* Z1 = Lg + B * m.k;   // hidden pre-activations       [B, h]
  float* DH = Z1 + (kHidden ? B * m.h : 0);  // hidden grad   [B, h]
  int* lab = reinterpret_cast<int*>(DH + (kHidden ? B * m.h : 0));  // [B]

  // entry offsets in the flat layout
  const int oW1 = 0;
  const int ob1 = kHidden ? m.d * m.h : 0;
  const int oW2 = kHidden ? ob1 + m.h : 0;
  const int ob2 = kHidden ? oW2 + m.h * m.k : m.d * m.k;

  for (int p = threadIdx.x; p < D; p += blockDim.x) {
    W[p] = theta_t[p];
    Dl[p] = 0.0f;
  }
  const int n = num_rows[c];
  const int64_t r0 = row_start[c];
  const int32_t* pc = perms + perm_off[c];
  const float* ctrl = control ? control + (int64_t)c * ld_control : nullptr;
  __syncthreads();

  for (int e = 0; e < epochs; ++e) {
    for (int start = 0; start < n; start += B) {
      const int nb = min(B, n - start);
      const int32_t* idx = pc + (int64_t)e * n + start;
      // gather the batch (coalesced along the feature axis)
      for (int t = threadIdx.x; t < nb * m.d; t += blockDim.x) {
        const int r = t / m.d, i = t - r * m.d;
        Xb[t] = X[(r0 + idx[r]) * m.d + i];
      }
      if (threadIdx.x < nb) lab[threadIdx.x] = y[r0 + idx[threadIdx.x]];
      __syncthreads();
      if constexpr (kHidden) {
        for (int t = threadIdx.x; t < nb * m.h; t += blockDim.x) {
          const int r = t / m.h, j = t - r * m.h;
          float z = W[ob1 + j];
          const float* xr = Xb + r * m.d;
          for (int i = 0; i < m.d; ++i) z = fmaf(xr[i], W[oW1 + i * m.h + j], z);
          Z1[t] = z;
        }
        __syncthreads();
      }
      for (int t = threadIdx.x; t < nb * m.k; t += blockDim.x) {
        const int r = t / m.k, q = t - r * m.k;
        float z = W[ob2 + q];
        for (int j = 0; j < hin; ++j) z = fmaf(act<kHidden>(Xb, Z1, m, r, j), W[oW2 + j * m.k + q], z);
        Lg[t] = z;
      }
      __syncthreads();
      // softmax cross-entropy gradient of the mean batch loss, one thread per row
      if (threadIdx.x < nb) {
        float* row = Lg + threadIdx.x * m.k;
        float mx = row[0];
        for (int q = 1; q < m.k; ++q) mx = fmaxf(mx, row[q]);
        float s = 0.0f;
        for (int q = 0; q < m.k; ++q) {
          row[q] = expf(row[q] - mx);
          s += row[q];
        }
        const int yl = lab[threadIdx.x];
        for (int q = 0; q < m.k; ++q) {
          float p = row[q] / s;
          if (q == yl) p -= 1.0f;
          row[q] = p / (float)nb;
        }
      }
      __syncthreads();
      // output layer gradient; hidden gradient (uses the pre-step W2)
      for (int t = threadIdx.x; t < hin * m.k; t += blockDim.x) {
        const int j = t / m.k, q = t - j * m.k;
        float g = 0.0f;
        for (int r = 0; r < nb; ++r) g = fmaf(act<kHidden>(Xb, Z1, m, r, j), Lg[r * m.k + q], g);
        G[oW2 + t] = g;
      }
      for (int q = threadIdx.x; q < m.k; q += blockDim.x) {
        float g = 0.0f;
        for (int r = 0; r < nb; ++r) g += Lg[r * m.k + q];
        G[ob2 + q] = g;
      }
      if constexpr (kHidden) {
        for (int t = threadIdx.x; t < nb * m.h; t += blockDim.x) {
          const int r = t / m.h, j = t - r * m.h;
          float g = 0.0f;
          for (int q = 0; q < m.k; ++q) g = fmaf(Lg[r * m.k + q], W[oW2 + j * m.k + q], g);
          DH[t] = Z1[t] > 0.0f ? g : 0.0f;
        }
        __syncthreads();
        for (int t = threadIdx.x; t < m.d * m.h; t += blockDim.x) {
          const int i = t / m.h, j = t - i * m.h;
          float g = 0.0f;
          for (int r = 0; r < nb; ++r) g = fmaf(Xb[r * m.d + i], DH[r * m.h + j], g);
          G[oW1 + t] = g;
        }
        for (int j = threadIdx.x; j < m.h; j += blockDim.x) {
          float g = 0.0f;
          for (int r = 0; r < nb; ++r) g += DH[r * m.h + j];
          G[ob1 + j] = g;
        }
      }
      __syncthreads();
      // theta <- theta - lr*(g + mu*(theta - theta_t) + c); theta - theta_t == -delta
      for (int p = threadIdx.x; p < D; p += blockDim.x) {
        float g = G[p];
        if (mu != 0.0f) g = fmaf(mu, -Dl[p], g);
        if (ctrl) g += ctrl[p];
        const float s = lr * g;
        W[p] -= s;
        Dl[p] += s;
      }
      __syncthreads();
    }
  }
  float* out = delta_out + (int64_t)c * ld_delta;
  int bad = 0;
  for (int p = threadIdx.x; p < D; p += blockDim.x) {
    const float v = Dl[p];
    bad |= !isfinite(v);
    out[p] = v;
  }
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) nonfinite[c] = bad;
}

template <bool kHidden>
__global__ void __launch_bounds__(kThreads) eval_small_kernel(
    const float* __restrict__ theta, Dims m, const float* __restrict__ X,
    const int32_t* __restrict__ y, const int64_t* __restrict__ row_start,
    const int32_t* __restrict__ num_rows, double* __restrict__ loss_sum,
    int32_t* __restrict__ correct) {
  extern __shared__ float smem[];
  __shared__ double red[32];
  const int c = blockIdx.x;
  const int D = m.D();
  const int hin = kHidden ? m.h : m.d;
  float* W = smem;
  float* Xc = W + D;                   // [R, d]
  float* Lg = Xc + kEvalRows * m.d;    // [R, k]
  float* Z1 = Lg + kEvalRows * m.k;    // [R, h]
  const int ob1 = kHidden ? m.d * m.h : 0;
  const int oW2 = kHidden ? ob1 + m.h : 0;
  const int ob2 = kHidden ? oW2 + m.h * m.k : m.d * m.k;
  for (int p = threadIdx.x; p < D; p += blockDim.x) W[p] = theta[p];
  const int n = num_rows[c];
  const int64_t r0 = row_start[c];
  double loss = 0.0;
  int hits = 0;
  __syncthreads();
  for (int start = 0; start < n; start += kEvalRows) {
    const int nr = min(kEvalRows, n - start);
    for (int t = threadIdx.x; t < nr * m.d; t += blockDim.x) Xc[t] = X[(r0 + start) * m.d + t];
    __syncthreads();
    if constexpr (kHidden) {
      for (int t = threadIdx.x; t < nr * m.h; t += blockDim.x) {
        const int r = t / m.h, j = t - r * m.h;
        float z = W[ob1 + j];
        for (int i = 0; i < m.d; ++i) z = fmaf(Xc[r * m.d + i], W[i * m.h + j], z);
        Z1[t] = z;
      }
      __syncthreads();
    }
    for (int t = threadIdx.x; t < nr * m.k; t += blockDim.x) {
      const int r = t / m.k, q = t - r * m.k;
      float z = W[ob2 + q];
      for (int j = 0; j < hin; ++j) z = fmaf(act<kHidden>(Xc, Z1, m, r, j), W[oW2 + j * m.k + q], z);
      Lg[t] = z;
    }
    __syncthreads();
    if (threadIdx.x < nr) {
      const float* row = Lg + threadIdx.x * m.k;
      float mx = row[0];
      int arg = 0;
      for (int q = 1; q < m.k; ++q)
        if (row[q] > mx) { mx = row[q]; arg = q; }  // first maximum, like numpy.argmax
      float s = 0.0f;
      for (int q = 0; q < m.k; ++q) s += expf(row[q] - mx);
      const int yl = y[r0 + start + threadIdx.x];
      loss += -((double)row[yl] - (double)mx - (double)logf(s));
      hits += (arg == yl);
    }
    __syncthreads();
  }
  const double tl = block_sum(loss, red);
  const double th = block_sum((double)hits, red);
  if (threadIdx.x == 0) {
    loss_sum[c] = tl;
    correct[c] = (int32_t)th;
  }
}

template <bool kHidden>
int launch_local_sgd(const float* theta_t, Dims m, const float* X, const int32_t* y,
                     const int64_t* row_start, const int32_t* num_rows, const int32_t* perms,
                     const int64_t* perm_off, int C, int epochs, int B, float lr, float mu,
                     const float* control, int64_t ld_control, float* delta_out, int64_t ld_delta,
                     int32_t* nonfinite, void* stream) {
  FB_REQUIRE(C >= 0 && epochs >= 0 && B >= 1, "local_sgd: bad cohort/epochs/batch (C=%d E=%d B=%d)", C, epochs, B);
  FB_REQUIRE(m.d >= 1 && m.k >= 1 && (!kHidden || m.h >= 1), "local_sgd: bad model dims");
  FB_REQUIRE(ld_delta >= m.D(), "local_sgd: ld_delta %lld < D %d", (long long)ld_delta, m.D());
  FB_REQUIRE(B <= kThreads, "local_sgd: batch_size %d > %d unsupported", B, kThreads);
  if (C == 0) return FB_OK;
  const size_t smem = sizeof(float) * (3 * (size_t)m.D() + (size_t)B * m.d + (size_t)B * m.k +
                                       (kHidden ? 2 * (size_t)B * m.h : 0)) + sizeof(int) * B;
  FB_UNSUPPORTED(smem <= 227 * 1024, "local_sgd: model needs %zu bytes of shared memory", smem);
  auto kern = local_sgd_small_kernel<kHidden>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  FB_LAUNCH(kHidden ? "local_sgd_mlp_kernel" : "local_sgd_linear_kernel", as_stream(stream), kern<<<C, kThreads, smem, as_stream(stream)>>>(theta_t, m, X, y, row_start, num_rows, perms,
                                                 perm_off, epochs, B, lr, mu, control, ld_control,
                                                 delta_out, ld_delta, nonfinite));
  return launch_status("local_sgd_small_kernel");
}

template <bool kHidden>
int launch_eval(const float* theta, Dims m, const float* X, const int32_t* y,
                const int64_t* row_start, const int32_t* num_rows, int C, double* loss_sum,
                int32_t* correct, void* stream) {
  FB_REQUIRE(C >= 0, "eval: negative cohort");
  FB_REQUIRE(m.d >= 1 && m.k >= 1 && (!kHidden || m.h >= 1), "eval: bad model dims");
  if (C == 0) return FB_OK;
  const size_t smem = sizeof(float) * ((size_t)m.D() + (size_t)kEvalRows * (m.d + m.k + (kHidden ? m.h : 0)));
  FB_UNSUPPORTED(smem <= 227 * 1024, "eval: model needs %zu bytes of shared memory", smem);
  auto kern = eval_small_kernel<kHidden>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  FB_LAUNCH(kHidden ? "eval_mlp_kernel" : "eval_linear_kernel", as_stream(stream), kern<<<C, kThreads, smem, as_stream(stream)>>>(theta, m, X, y, row_start, num_rows, loss_sum, correct));
  return launch_status("eval_small_kernel");
}

}  // namespace
}  // namespace fb

extern "C" {

int fb_eval_linear_f32(const float* theta, int dim, int num_classes, const float* X,
                       const int32_t* y, const int64_t* row_start, const int32_t* num_rows,
                       int num_clients, double* loss_sum, int32_t* correct, void* stream) {
  return fb::launch_eval<false>(theta, fb::Dims{dim, 0, num_classes}, X, y, row_start, num_rows,
                                num_clients, loss_sum, correct, stream);
}

int fb_eval_mlp_f32(const float* theta, int dim, int hidden, int num_classes, const float* X,
                    const int32_t* y, const int64_t* row_start, const int32_t* num_rows,
                    int num_clients, double* loss_sum, int32_t* correct, void* stream) {
  return fb::launch_eval<true>(theta, fb::Dims{dim, hidden, num_classes}, X, y, row_start,
                               num_rows, num_clients, loss_sum, correct, stream);
}

int fb_local_sgd_linear_f32(const float* theta_t, int dim, int num_classes, const float* X,
                            const int32_t* y, const int64_t* row_start, const int32_t* num_rows,
                            const int32_t* perms, const int64_t* perm_off, int num_clients,
                            int epochs, int batch_size, float lr, float prox_mu,
                            const float* control, int64_t ld_control, float* delta_out,
                            int64_t ld_delta, int32_t* nonfinite, void* stream) {
  return fb::launch_local_sgd<false>(theta_t, fb::Dims{dim, 0, num_classes}, X, y, row_start,
                                     num_rows, perms, perm_off, num_clients, epochs, batch_size,
                                     lr, prox_mu, control, ld_control, delta_out, ld_delta,
                                     nonfinite, stream);
}

int fb_local_sgd_mlp_f32(const float* theta_t, int dim, int hidden, int num_classes,
                         const float* X, const int32_t* y, const int64_t* row_start,
                         const int32_t* num_rows, const int32_t* perms, const int64_t* perm_off,
                         int num_clients, int epochs, int batch_size, float lr, float prox_mu,
                         const float* control, int64_t ld_control, float* delta_out,
                         int64_t ld_delta, int32_t* nonfinite, void* stream) {
  return fb::launch_local_sgd<true>(theta_t, fb::Dims{dim, hidden, num_classes}, X, y,
                                    row_start, num_rows, perms, perm_off, num_clients, epochs,
                                    batch_size, lr, prox_mu, control, ld_control, delta_out,
                                    ld_delta, nonfinite, stream);
}

}  // extern "C"
