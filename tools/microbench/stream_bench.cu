// HBM streaming read rate vs per-SM concurrency on B200: how many warps and
// loads in flight one SM needs to pull its share of HBM bandwidth.  Informs
// the warp split of clip_aggregate_fused.cu (norm warps stream HBM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bench stream_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NB>
__global__ void stream_sum(const float4* __restrict__ x, long long n4, int active_threads, double* out) {
  if (threadIdx.x >= active_threads) return;
  // each CTA owns a contiguous slice (like the fused kernel)
  const long long per = (n4 + gridDim.x - 1) / gridDim.x;
  const long long lo = blockIdx.x * per, hi = lo + per < n4 ? lo + per : n4;
  float acc = 0.f;
  for (long long i = lo + threadIdx.x; i < hi; i += (long long)active_threads * NB) {
    float4 v[NB];
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const long long j = i + (long long)q * active_threads;
      v[q] = j < hi ? __ldcs(x + j) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int q = 0; q < NB; ++q) acc += v[q].x + v[q].y + v[q].z + v[q].w;
  }
  if (acc == 12345.f) *out = acc;
}

template <int NB>
void run(const float4* x, long long n4, int blocks, int threads, int active, double* out) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 2; ++w) stream_sum<NB><<<blocks, threads>>>(x, n4, active, out);
  cudaEventRecord(a);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) stream_sum<NB><<<blocks, threads>>>(x, n4, active, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double gbs = (double)n4 * 16 * reps / (ms * 1e-3) / 1e9;
  printf("blocks %4d threads %4d active %4d loads/thread %2d  in-flight/SM %6.0f KB  %7.1f GB/s\n", blocks, threads,
         active, NB, (double)active * NB * 16 * blocks / 148 / 1024, gbs);
}

int main_plain() {
  const long long bytes = 4LL << 30;  // 4 GB >> L2
  const long long n4 = bytes / 16;
  float4* x;
  double* out;
  cudaMalloc(&x, bytes);
  cudaMalloc(&out, 8);
  cudaMemset(x, 0, bytes);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<2>(x, n4, sms * 8, 256, 256, out);
  run<4>(x, n4, sms * 4, 256, 256, out);
  run<8>(x, n4, sms, 256, 256, out);
  run<16>(x, n4, sms, 256, 256, out);
  run<32>(x, n4, sms, 256, 256, out);
  run<8>(x, n4, sms, 512, 512, out);
  run<16>(x, n4, sms, 512, 512, out);
  run<16>(x, n4, sms, 512, 256, out);
  run<32>(x, n4, sms, 512, 256, out);
  run<8>(x, n4, sms, 1024, 1024, out);
  run<4>(x, n4, sms, 1024, 1024, out);
  run<4>(x, n4, sms * 2, 1024, 1024, out);
  return 0;
}

// ---- bulk-copy (cp.async.bulk) ring: 1 producer thread per SM streams its contiguous slice
// into a STAGES x CHUNK shared-memory ring, NW consumer warps read it (sum of squares, fp64).
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int STAGES, int CHUNK, int NW>
__global__ void __launch_bounds__((NW + 1) * 32, 1) bulk_stream(const float* __restrict__ x, long long n, double* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const long long per = ((n + gridDim.x - 1) / gridDim.x + 3) & ~3LL;
  const long long lo = blockIdx.x * per, hi = lo + per < n ? lo + per : n;
  const int nchunks = hi > lo ? (int)(((hi - lo) * 4 + CHUNK - 1) / CHUNK) : 0;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(NW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == NW) {  // producer
    if ((threadIdx.x & 31) == 0) {
      for (int c = 0; c < nchunks; ++c) {
        const int s = c % STAGES;
        const uint32_t ph = (c / STAGES) & 1;
        if (c >= STAGES) {
          asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su32(&empty[s])), "r"(ph ^ 1) : "memory");
        }
        const long long off = lo * 4 + (long long)c * CHUNK;
        const uint32_t bytes = (uint32_t)((hi * 4 - off) < CHUNK ? (hi * 4 - off) : CHUNK);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(smem + s * CHUNK)),
                     "l"((const char*)x + off), "r"(bytes), "r"(su32(&full[s])) : "memory");
      }
    }
    return;
  }
  double acc = 0.0;
  for (int c = 0; c < nchunks; ++c) {
    const int s = c % STAGES;
    const uint32_t ph = (c / STAGES) & 1;
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su32(&full[s])), "r"(ph) : "memory");
    const float4* b = reinterpret_cast<const float4*>(smem + s * CHUNK);
    const long long off = lo * 4 + (long long)c * CHUNK;
    const int nf4 = (int)(((hi * 4 - off) < CHUNK ? (hi * 4 - off) : CHUNK) / 16);
    for (int i = threadIdx.x; i < nf4; i += NW * 32) {
      const float4 v = b[i];
      acc += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
  }
  if (acc == 12345.0) *out = acc;
}

template <int STAGES, int CHUNK, int NW>
void run_bulk(const float* x, long long n, double* out) {
  auto k = bulk_stream<STAGES, CHUNK, NW>;
  const int smem = STAGES * CHUNK;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<<<148, (NW + 1) * 32, smem>>>(x, n, out);
  k<<<148, (NW + 1) * 32, smem>>>(x, n, out);
  cudaEventRecord(a);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) k<<<148, (NW + 1) * 32, smem>>>(x, n, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("bulk ring %d x %6d B, %2d consumer warps: %7.1f GB/s  (%s)\n", STAGES, CHUNK, NW,
         (double)n * 4 * reps / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main_bulk() {
  const long long bytes = 4LL << 30;
  float* x;
  double* out;
  cudaMalloc(&x, bytes);
  cudaMalloc(&out, 8);
  cudaMemset(x, 0, bytes);
  const long long n = bytes / 4;
  run_bulk<4, 16384, 8>(x, n, out);
  run_bulk<8, 16384, 8>(x, n, out);
  run_bulk<4, 32768, 8>(x, n, out);
  run_bulk<6, 32768, 8>(x, n, out);
  run_bulk<6, 32768, 16>(x, n, out);
  run_bulk<3, 32768, 16>(x, n, out);
  run_bulk<12, 16384, 16>(x, n, out);
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1) return main_bulk();
  return main_plain();
}
