// microbenchmark: kind::f16 MMA issue rate with MN-major operands in the
// conv2 weight-gradient pattern (A: a1 positions x 32 ci, SWIZZLE_64B, the
// M blocks one position apart; B: dz2 [hi | lo] SWIZZLE_128B, N = 128 + 64)
// against the same MMAs with K-major operands (tools/microbench)
#include <cstdio>
#include <cuda.h>
#include "../../paper_2404_06430_b200/csrc/tc_common.cuh"
using namespace fb;
template <bool MN>
__global__ void __launch_bounds__(128, 1) kern(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  tc::fence_proxy_async();
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&tslot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t ah = tc::smem_u32(sm), al = ah + 20480, bh = ah + 40960;  // B hi | lo 30720 apart
    constexpr uint32_t I2 = MN ? tc::idesc_f16_mn(128, 128) : tc::idesc_f16(128, 128);
    constexpr uint32_t I1 = MN ? tc::idesc_f16_mn(128, 64) : tc::idesc_f16(128, 64);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll 5
      for (int ks = 0; ks < 15; ++ks) {
        uint64_t adh, adl, bdh;
        if (MN) {
          adh = tc::sdesc(ah + ks * 16 * 64, 64, 512, 4);
          adl = tc::sdesc(al + ks * 16 * 64, 64, 512, 4);
          bdh = tc::sdesc(bh + ks * 16 * 128, 30720, 1024, 2);
        } else {
          adh = tc::sdesc(ah + (ks & 1) * 32, 16, 512, 4);
          adl = tc::sdesc(al + (ks & 1) * 32, 16, 512, 4);
          bdh = tc::sdesc(bh + (ks & 1) * 32, 16, 512, 4);
        }
        tc::mma2_f16(tmem, tmem + 128, adh, adl, bdh, I2, I1, 1);
      }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(tmem);
}
template <bool MN>
void run(const char* name) {
  long long* d; cudaMalloc(&d, 148 * 8);
  auto k = kern<MN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
  const int iters = 400;
  k<<<148, 128, 170 * 1024>>>(d, iters);
  k<<<148, 128, 170 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  printf("%-12s %.1f clk per K step (N=128 + N=64 MMA pair; K-major SS measured 64 + 48)  err=%s\n", name,
         avg / (iters * 15.0), cudaGetErrorString(e));
  cudaFree(d);
}
int main() {
  run<false>("K-major");
  run<true>("MN-major");
  return 0;
}
