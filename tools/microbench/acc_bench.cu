// How accurate is fp32 accumulation in TMEM over long tcgen05.mma chains? (tools/microbench)
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda.h>
#include <cuda_fp16.h>
#include "../../paper_2404_06430_b200/csrc/tc_common.cuh"
using namespace fb;
// A: L tiles of [128 rows][16 k] fp16 K-major SW32?  Use no-swizzle-free layout: SW64 with 32-B used per row
// Simpler: K-major SWIZZLE_64B tiles of 128 x 32 fp16 (2 k-steps per tile)
__device__ __forceinline__ uint32_t sw64(uint32_t row, uint32_t k) { return row * 64u + ((((k >> 3) ^ ((row >> 1) & 3u)) << 4) | ((k & 7u) << 1)); }
__global__ void __launch_bounds__(128, 1) kern(const __half* A, const __half* B, int L, float* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int T = (L + 1) / 2;  // tiles of 32 k
  uint8_t* sA = sm;                 // T x 8 KB
  uint8_t* sB = sm + T * 8192;      // T x 4 KB (64 rows)
  for (int i = threadIdx.x; i < T * 128 * 32; i += blockDim.x) {
    const int t = i / (128 * 32), r = (i / 32) % 128, k = i % 32;
    *reinterpret_cast<__half*>(sA + t * 8192 + sw64(r, k)) = A[i];
  }
  for (int i = threadIdx.x; i < T * 64 * 32; i += blockDim.x) {
    const int t = i / (64 * 32), r = (i / 32) % 64, k = i % 32;
    *reinterpret_cast<__half*>(sB + t * 4096 + sw64(r, k)) = B[i];
  }
  tc::fence_proxy_async();
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc<64>(&tslot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    for (int s = 0; s < L; ++s) {
      const uint32_t a = tc::smem_u32(sA + (s / 2) * 8192) + 32 * (s & 1);
      const uint32_t b = tc::smem_u32(sB + (s / 2) * 4096) + 32 * (s & 1);
      tc::mma_f16(tmem, tc::sdesc(a, 16, 512, 4), tc::sdesc(b, 16, 512, 4), tc::idesc_f16(128, 64), s > 0);
    }
    tc::mma_commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  const int w = threadIdx.x >> 5;
  uint32_t v[32];
  for (int h = 0; h < 2; ++h) {
    tc::tmem_ld32(tmem + ((uint32_t)(w * 32) << 16) + h * 32, v);
    tc::tmem_ld_wait();
    for (int j = 0; j < 32; ++j) out[(w * 32 + (threadIdx.x & 31)) * 64 + h * 32 + j] = __uint_as_float(v[j]);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x < 32) tc::tmem_dealloc<64>(tmem);
}
int main() {
  srand(1);
  for (int L : {2, 6, 18, 36, 100}) {
    const int T = (L + 1) / 2;
    std::vector<__half> A(T * 128 * 32), B(T * 64 * 32);
    std::vector<float> Af(A.size()), Bf(B.size());
    for (size_t i = 0; i < A.size(); ++i) { float x = ((rand() / (float)RAND_MAX) * 2 - 1) * 16384.f; A[i] = __float2half(x); Af[i] = __half2float(A[i]); }
    for (size_t i = 0; i < B.size(); ++i) { float x = ((rand() / (float)RAND_MAX)) * 16384.f; B[i] = __float2half(x); Bf[i] = __half2float(B[i]); }
    __half *dA, *dB; float* dO;
    cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dO, 128 * 64 * 4);
    cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    const int smem = T * 12288 + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<1, 128, smem>>>(dA, dB, L, dO);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> O(128 * 64);
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    double maxrel = 0, sumrel = 0, bias = 0, maxrel_mag = 0; int n = 0;
    double fp32err = 0;
    for (int r = 0; r < 128; ++r) for (int c = 0; c < 64; ++c) {
      double exact = 0, mag = 0; float f32 = 0;
      for (int s = 0; s < L; ++s) for (int k = 0; k < 16; ++k) {
        const int t = s / 2, kk = (s & 1) * 16 + k;
        const double p = (double)Af[(t * 128 + r) * 32 + kk] * Bf[(t * 64 + c) * 32 + kk];
        exact += p; mag += fabs(p); f32 += (float)p;
      }
      const double err = O[r * 64 + c] - exact;
      maxrel = fmax(maxrel, fabs(err) / mag); sumrel += fabs(err) / mag; bias += err / mag; ++n;
      fp32err += fabs((double)f32 - exact) / mag;
    }
    printf("L=%3d MMAs (%4d products): TC err/sum|p|: max %.2e mean %.2e bias %.2e | sequential fp32 mean %.2e  (%s)\n",
           L, L * 16, maxrel, sumrel / n, bias / n, fp32err / n, cudaGetErrorString(e));
  }
}
