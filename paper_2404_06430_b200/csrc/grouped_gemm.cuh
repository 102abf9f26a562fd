// The grouped (per-client) fp32 GEMM of lm.cu, shared with resnet.cu: one launch
// computes C[z] = alpha A[z] B[z] (+ beta C[z]) (+ bias[z]) for every client z of
// a wave, on the tcgen05 3xTF32 persistent kernel when the operands are TMA-legal
// (16-byte aligned bases and strides, M, N >= 64) and on the SIMT tiled kernel
// otherwise.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fb {
namespace lm {

// C[z](m, n) = alpha * sum_k A[z](m, k) B[z](k, n) (+ beta C) (+ bias[z](n)),
//   A(m, k) = TA ? A[k * lda + m] : A[m * lda + k]   (relu_a: max(0, .))
//   B(k, n) = TB ? B[n * ldb + k] : B[k * ldb + n]   (relu_b: max(0, .))
// mask_aux: multiply the result by (aux[z](m, n) > 0)  (ReLU backward).
// Batches (clients) whose active[z] == 0 are skipped.
struct Gemm {
  const float* A;
  int64_t lda, sA;
  const float* B;
  int64_t ldb, sB;
  float* C;
  int64_t ldc, sC;
  int M, N, K;
  const float* bias;
  int64_t sBias;
  const float* aux;
  int64_t ldaux, sAux;
  const int32_t* active;
  float alpha, beta;
  int relu_a, relu_b;
};

Gemm gemm_base();
// family: launch-label set (0 = lm_gemm_*, 1 = rn_gemm_*)
int launch_gemm(bool TA, bool TB, const Gemm& g, int batch, cudaStream_t s, int family = 0);
extern int g_gemm_impl;  // 1 = tcgen05 3xTF32 (default), 0 = SIMT FP32

}  // namespace lm
}  // namespace fb
