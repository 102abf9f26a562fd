// tcgen05.mma kind::f16 issue rate with A in TMEM (.ts) vs both operands in SMEM (tools/microbench)
#include <cstdio>
#include <cuda.h>
#include "../../paper_2404_06430_b200/csrc/tc_common.cuh"
using namespace fb;
template <int N, int TS>
__global__ void __launch_bounds__(128, 1) kern(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 196 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  tc::fence_proxy_async();
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&tslot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {
    if (tc::elect_one()) {
      constexpr uint32_t idesc = tc::idesc_f16(128, N);
      const uint32_t s0 = tc::smem_u32(sm);
      long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
          const uint32_t b = s0 + (it & 3) * 16384 + ((tap / 3) * 30 + tap % 3) * 64;
          const uint64_t bd = tc::sdesc(b, 16, 512, 4);
          if (TS) {
            const uint32_t a = tmem + 256 + tap * 16;
            asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;" ::"r"(tmem), "r"(a), "l"(bd),
                         "r"(idesc) : "memory");
          } else {
            const uint64_t ad = tc::sdesc(s0 + 65536 + tap * 4096, 16, 512, 4);
            tc::mma_f16(tmem, ad, bd, idesc, 1);
          }
        }
      }
      tc::mma_commit(&bar);
      tc::mbar_wait(&bar, 0);
      out[blockIdx.x] = clock64() - t0;
    }
    __syncwarp();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(tmem);
}
template <int N, int TS>
void run(const char* name) {
  long long* d; cudaMalloc(&d, 148 * 8);
  auto k = kern<N, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int iters = 1000;
  k<<<148, 128, 200 * 1024>>>(d, iters);
  k<<<148, 128, 200 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  printf("%-10s N=%3d: %.1f clk/MMA (floor %d)  %s\n", name, N, avg / (iters * 9), 128 * N / 256, cudaGetErrorString(e));
}
int main() { run<64, 0>("SS"); run<128, 0>("SS"); run<64, 1>("TS"); run<128, 1>("TS"); run<256, 1>("TS"); return 0; }
