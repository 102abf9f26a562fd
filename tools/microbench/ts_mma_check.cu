// Correctness probe: tcgen05.mma kind::f16 with A from TMEM (".ts": A written with
// tcgen05.st as packed fp16 pairs, lane = row) vs a CPU reference.  (tools/microbench)
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda.h>
#include <cuda_fp16.h>
#include "../../paper_2404_06430_b200/csrc/tc_common.cuh"
using namespace fb;
__device__ __forceinline__ uint32_t sw64(uint32_t row, uint32_t k) { return row * 64u + ((((k >> 3) ^ ((row >> 1) & 3u)) << 4) | ((k & 7u) << 1)); }
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
}
template <int N>
__global__ void __launch_bounds__(128, 1) kern(const __half* A, const __half* B, int K, float* out) {
  __shared__ __align__(1024) uint8_t sB[N * 64 * 2];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__half*>(sB + (k / 32) * N * 64 + sw64(r, k % 32)) = B[i];
  }
  tc::fence_proxy_async();
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc<256>(&tslot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t acol = 128;  // A columns start here (K/2 of them)
  {
    const int r = warp * 32 + lane;
    for (int j0 = 0; j0 < K / 2; j0 += 8) {
      uint32_t v[8];
      for (int j = 0; j < 8; ++j) {
        const __half lo = A[r * K + 2 * (j0 + j)], hi = A[r * K + 2 * (j0 + j) + 1];
        v[j] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
      }
      tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + acol + j0, v);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = tc::idesc_f16(128, N);
    for (int ks = 0; ks < K / 16; ++ks) {
      const uint32_t b = tc::smem_u32(sB) + (ks / 2) * N * 64 + (ks & 1) * 32;
      const uint64_t bd = tc::sdesc(b, 16, 512, 4);
      const uint32_t a = tmem + acol + ks * 8;
      const uint32_t acc = ks > 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem), "r"(a), "l"(bd),
                   "r"(idesc), "r"(acc) : "memory");
    }
    tc::mma_commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
    tc::tmem_ld_wait();
    for (int j = 0; j < 32; ++j) out[(warp * 32 + lane) * N + c0 + j] = __uint_as_float(v[j]);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 0) tc::tmem_dealloc<256>(tmem);
}
template <int N>
void run(int K) {
  std::vector<__half> A(128 * K), B(N * K);
  std::vector<float> Af(A.size()), Bf(B.size());
  for (size_t i = 0; i < A.size(); ++i) { A[i] = __float2half((rand() % 2001 - 1000) / 256.f); Af[i] = __half2float(A[i]); }
  for (size_t i = 0; i < B.size(); ++i) { B[i] = __float2half((rand() % 2001 - 1000) / 256.f); Bf[i] = __half2float(B[i]); }
  __half *dA, *dB; float* dO;
  cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dO, 128 * N * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  kern<N><<<1, 128>>>(dA, dB, K, dO);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> O(128 * N);
  cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int r = 0; r < 128; ++r) for (int n = 0; n < N; ++n) {
    double s = 0; for (int k = 0; k < K; ++k) s += (double)Af[r * K + k] * Bf[n * K + k];
    maxerr = fmax(maxerr, fabs(s - O[r * N + n]));
  }
  printf("TS MMA N=%d K=%d: max abs err %.3e (%s)\n", N, K, maxerr, cudaGetErrorString(e));
}
int main() { run<64>(16); run<64>(32); run<128>(64); run<64>(128); return 0; }
