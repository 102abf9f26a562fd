// microbenchmark: tcgen05.mma kind::f16 issue rate for small N (tools/microbench)
#include <cstdio>
#include <cuda.h>
#include "../../paper_2404_06430_b200/csrc/tc_common.cuh"
using namespace fb;
template <int N, int LAYOUT, int PATTERN, int RND = 0>
__global__ void __launch_bounds__(128, 1) kern(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x * 97u; h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    // two fp16 in [-2^14, 2^14) with random mantissas (sign, exponent 10..28)
    uint32_t v = ((h & 0x83ffu) | (((h >> 10) % 18 + 10) << 10));
    uint32_t w = (((h >> 16) & 0x83ffu) | ((((h >> 20) % 18) + 10) << 10));
    reinterpret_cast<uint32_t*>(sm)[i] = RND ? (v | (w << 16)) : 0;
  }
  tc::fence_proxy_async();
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&tslot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = tc::idesc_f16(128, N);
    const uint32_t a = tc::smem_u32(sm), b = a + 32768;
    const uint32_t sbo = LAYOUT == 4 ? 512 : 1024;
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int k = 0; k < 2; ++k) {
        const uint64_t ad = tc::sdesc(a + 32 * k + (PATTERN == 3 ? (it % 9) * 64 : 0), 16, sbo, LAYOUT);
        const uint64_t bd = tc::sdesc(b + 32 * k, 16, sbo, LAYOUT);
        if (PATTERN == 0) tc::mma_f16(tmem, ad, bd, idesc, 1);
        else {
          tc::mma_f16(tmem, ad, bd, idesc, 1);
          tc::mma_f16(tmem + 256, ad, bd, idesc, 1);
          tc::mma_f16(tmem + 256, ad, bd, idesc, 1);
        }
      }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(tmem);
}
template <int N, int L, int P, int R = 0>
void run(const char* name) {
  long long* d; cudaMalloc(&d, 148 * 8);
  auto k = kern<N, L, P, R>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  const int iters = 2000;
  k<<<148, 128, 66 * 1024>>>(d, iters);
  k<<<148, 128, 66 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  const int mmas = iters * 2 * (P == 0 ? 1 : 3);
  printf("%-40s N=%3d: %.1f clk/MMA (floor %d)  err=%s\n", name, N, avg / mmas, 128 * N / 256, cudaGetErrorString(e));
  cudaFree(d);
}
int main() {
  run<64, 4, 1, 0>("3-MMA SW64 zeros");
  run<64, 4, 1, 1>("3-MMA SW64 random");
  run<128, 4, 0, 0>("single SW64 zeros");
  run<128, 4, 0, 1>("single SW64 random");
  run<256, 4, 0, 1>("single SW64 random");
  run<32, 2, 1, 1>("3-MMA SW128 random");
  return 0;
}
