// microbenchmark: tcgen05.mma kind::f16 with the conv2 forward's real operand walk (tools/microbench)
#include <cstdio>
#include <cuda.h>
#include "../../paper_2404_06430_b200/csrc/tc_common.cuh"
using namespace fb;
template <int N, int WALK>
__global__ void __launch_bounds__(128, 1) kern(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  tc::fence_proxy_async();
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&tslot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = tc::idesc_f16(128, N);
    const uint32_t sB0 = tc::smem_u32(sm), sA0 = sB0 + 73728;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int stage = WALK >= 1 ? it & 3 : 0;
      for (int tap = 0; tap < 9; ++tap) {
        const uint32_t ah = sA0 + stage * 28672 + (WALK >= 2 ? ((tap / 3) * 30 + tap % 3) * 64 : 0), al = ah + 14336;
        const uint32_t bh = sB0 + (WALK >= 1 ? tap * 2 * N * 64 : 0), bl = bh + N * 64;
        const uint32_t dmain = tmem + (tap / 3) * N, dcross = tmem + 3 * N;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const uint64_t adh = tc::sdesc(ah + 32 * k, 16, 512, 4), adl = tc::sdesc(al + 32 * k, 16, 512, 4);
          const uint64_t bdh = tc::sdesc(bh + 32 * k, 16, 512, 4), bdl = tc::sdesc(bl + 32 * k, 16, 512, 4);
          tc::mma_f16(dmain, adh, bdh, idesc, 1);
          tc::mma_f16(dcross, adh, bdl, idesc, 1);
          tc::mma_f16(dcross, adl, bdh, idesc, 1);
        }
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
template <int N, int W>
void run(const char* name) {
  long long* d; cudaMalloc(&d, 148 * 8);
  auto k = kern<N, W>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 202 * 1024);
  const int iters = 400;
  k<<<148, 128, 202 * 1024>>>(d, iters);
  k<<<148, 128, 202 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  printf("%-44s N=%d: %.1f clk/MMA  err=%s\n", name, N, avg / (iters * 54), cudaGetErrorString(e));
}
int main() {
  run<64, 0>("fixed A, fixed B");
  run<64, 1>("stage walk + per-tap B");
  run<64, 2>("stage walk + per-tap B + row-shifted A");
  return 0;
}
