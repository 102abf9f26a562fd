// K2 + K3 fused: per-client L2 norm, clip factor and the weighted sum in ONE
// HBM pass over the [C, ld] delta matrix.
//
// The clip factor of client c needs the norm of its whole row before any of
// its columns can be summed (fedsim/privacy/clipping.py:37-56, then
// fedsim/engine/aggregator.py:39-44), so a two-kernel K2 -> K3 design reads
// every row twice from HBM and caps at ~50 % of the algorithmic roofline
// B_alg = 4*D*C.  This kernel reads each row from
// HBM once:
//
// * One persistent cooperative CTA per SM owns a fixed, contiguous column
//   slice (rows of 2048 floats; 33 rows per SM at D = 10 M) and keeps the
//   running aggregate of that slice ON CHIP -- in TENSOR MEMORY (256 KB per
//   SM = 32 slice rows, read-modify-written with tcgen05.ld / tcgen05.st) plus
//   2 overflow rows in shared memory: 10.3 M columns on 148 SMs.  TMEM is
//   otherwise idle here; as the accumulator it leaves registers and shared
//   memory to the data streams.
// * Two producer warps drive two cp.async.bulk rings (global -> shared,
//   3 x 32 KB stages of 4 slice rows each, mbarrier complete_tx):
//     norm ring: every client's slice from HBM (L2 policy evict_last);
//     acc ring : the same slices again, one client behind, re-read from L2
//                where the norm ring left them (two 40 MB rows of a 10 M-
//                parameter model fit the 126 MB L2), policy evict_first.
//   The copy engine keeps the bytes in flight without holding registers
//   (tools/microbench/stream_bench.cu: such a ring streams HBM at >= 6.7 TB/s
//   from 8 consumer warps, where 8 warps of plain loads stop near 4 TB/s).
// * Two consumer groups of 8 warps run CONCURRENTLY:
//     norm group: squares of client k (fp64) -> the CTA's partial[k, b],
//       published with a release increment of counter[k].  It never waits on
//       other CTAs, only stays at most one client (two when D <= 5.3 M) ahead
//       of its own accumulate group, bounding the clients live in L2;
//     accumulate group: waits (acquire) until counter[k] == grid size, derives
//       coef[k] from the G partials in a fixed order (the same bits in every
//       CTA), and adds coef[k] * client k into the TMEM / smem accumulators.
//   A slow CTA therefore delays the others' accumulation by up to a client,
//   not their HBM stream.  (A single consumer group alternating norm and
//   accumulate phases measured 0.55 of the roofline, stalled on that wait.)
//
// Every 64 clients the fp32 accumulators are added into an fp64 global
// accumulator (8 bytes per column per 64 clients: < 4 % extra traffic), so
// the sum stays within ~1e-7 of the fp64 two-pass path; results are
// bit-identical run to run (fixed per-element order: clients in queue order).

#include "fb_common.cuh"
#include "tc_common.cuh"

namespace fb {
namespace {

constexpr int kGroup = 256;                      // threads per consumer group (8 warps)
constexpr int kT = 64 + 2 * kGroup;              // 2 producer warps + norm consumers + acc consumers
constexpr int kRowF = 2048;                      // floats per slice row: two float4 per consumer thread
constexpr int kRowsPerStage = 4;
constexpr int kStageBytes = kRowsPerStage * kRowF * 4;  // 32 KB
constexpr int kTmemRows = 32;                    // 256 TMEM columns per acc-consumer thread / 8
constexpr int kSmemRows = 2;                     // overflow accumulator rows in shared memory
constexpr int kMaxRows = kTmemRows + kSmemRows;
constexpr int kFlush = 64;                       // clients per fp32 accumulation block
constexpr long long kSpinLimit = 20LL * 1000 * 1000 * 1000;  // ~10 s of SM clocks
template <int kNormStages, int kAccStages>
constexpr size_t smem_bytes() {
  return (size_t)(kNormStages + kAccStages) * kStageBytes + sizeof(float) * kRowF * kSmemRows + 1024;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 1-D bulk copy global -> shared with an L2 cache policy
__device__ __forceinline__ void bulk_load_hint(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                               uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  const uint32_t a = tc::smem_u32(bar);
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void bar_group(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(kGroup) : "memory"); }
// TMEM: 32 lanes x 32 consecutive fp32 columns (4 slice rows x two float4 of one thread)
__device__ __forceinline__ void tmem_ld32f(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  tc::tmem_ld32(taddr, r);
  tc::tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st32f(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
      "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
      "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}
// TMEM: 32 lanes x 16 consecutive fp32 columns (4 slice rows of one thread's float4)
__device__ __forceinline__ void tmem_ld16f(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  tc::tmem_ld16(taddr, r);
  tc::tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st16f(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ double sq4(float4 v) {
  return (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
}
// zero the lanes of a float4 at column col that lie at or beyond D
__device__ __forceinline__ float4 mask_tail(float4 v, int64_t col, int64_t D) {
  if (col + 3 < D) return v;
  if (col + 0 >= D) v.x = 0.f;
  if (col + 1 >= D) v.y = 0.f;
  if (col + 2 >= D) v.z = 0.f;
  if (col + 3 >= D) v.w = 0.f;
  return v;
}

struct Args {
  const float* delta;
  const int32_t* rows;  // nullable: client k's update is delta row rows[k] (else row k)
  int64_t ld;
  int C;
  int64_t D;
  const float* w;
  double bound;
  double* norm;
  float* coef;
  int32_t* clipped;
  int32_t* nonfinite;
  float* agg;
  int accumulate;
  double* partial;    // [C, G]
  unsigned* counter;  // [C], zero on entry
  double* agg64;      // [D] fp64 block accumulator (only when C > kFlush)
  int lead;           // clients the norm group may run ahead of the accumulate group
};

// CTA-scope acquire load / release store of a shared flag: race-free (unlike a volatile
// access) and, unlike an atomic RMW spin, no serialised shared atomics from the 256 spinning
// threads of the norm group (atomicAdd(&flag, 0) cost ~7% of the step: 0.675 -> 0.63 of B_alg)
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(tc::smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(p)), "r"(v) : "memory");
}

template <int kNormStages, int kAccStages>
__global__ void __launch_bounds__(kT, 1) clip_aggregate_fused_kernel(const Args a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* norm_ring = smem;
  unsigned char* acc_ring = smem + kNormStages * kStageBytes;
  float4* sacc = reinterpret_cast<float4*>(acc_ring + kAccStages * kStageBytes);  // [kSmemRows][kRowF / 4]
  __shared__ __align__(8) uint64_t norm_full[kNormStages], norm_empty[kNormStages];
  __shared__ __align__(8) uint64_t acc_full[kAccStages], acc_empty[kAccStages];
  __shared__ uint32_t tmem_base;
  __shared__ double red[2][kGroup / 32];  // norm partials per warp, double-buffered by client parity
  __shared__ float s_cf;
  __shared__ int acc_done;                 // clients fully accumulated by this CTA (acquire / release access)

  const int G = gridDim.x, b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t R = (a.D + kRowF - 1) / kRowF;
  const int64_t rbase = R / G, rextra = R % G;
  const int64_t r0 = b * rbase + (b < rextra ? b : rextra);
  const int nr = (int)(rbase + (b < rextra ? 1 : 0));
  const int nst = nr > 0 ? (nr + kRowsPerStage - 1) / kRowsPerStage : 0;  // stages per client
  const int64_t slice_lo = r0 * kRowF;                                       // first column of the slice
  const int64_t slice_hi = (r0 + nr) * kRowF < a.ld ? (r0 + nr) * kRowF : a.ld;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kNormStages; ++s) {
      tc::mbar_init(&norm_full[s], 1);
      tc::mbar_init(&norm_empty[s], kGroup / 32);
    }
    for (int s = 0; s < kAccStages; ++s) {
      tc::mbar_init(&acc_full[s], 1);
      tc::mbar_init(&acc_empty[s], kGroup / 32);
    }
    tc::fence_mbar_init();
    atomicExch(&acc_done, 0);
  }
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();

  if (warp < 2) {
    // --------------------------------------------------------------- producers
    // warp 0 streams every client's slice into the norm ring, warp 1 every client's slice
    // (again, one client behind, from L2) into the acc ring; each runs ahead of the consumers
    // by its ring depth, independently of the other
    if (lane == 0 && nst > 0) {
      const bool norm_side = warp == 0;
      const uint64_t pol = norm_side ? policy_evict_last() : policy_evict_first();
      const int stages = norm_side ? kNormStages : kAccStages;
      unsigned char* ring = norm_side ? norm_ring : acc_ring;
      uint64_t* full = norm_side ? norm_full : acc_full;
      uint64_t* empty = norm_side ? norm_empty : acc_empty;
      int i = 0;
      for (int k = 0; k < a.C; ++k) {
        for (int s = 0; s < nst; ++s, ++i) {
          const int64_t c0 = slice_lo + (int64_t)s * kRowsPerStage * kRowF;
          const int64_t left = slice_hi - c0;
          const uint32_t bytes = (uint32_t)(4 * (left < kRowsPerStage * kRowF ? left : kRowsPerStage * kRowF));
          const int slot = i % stages;
          if (i >= stages) mbar_wait_spin(&empty[slot], ((i / stages) - 1) & 1);
          tc::mbar_arrive_expect_tx(&full[slot], bytes);
          const int64_t row = a.rows ? (int64_t)__ldg(a.rows + k) : (int64_t)k;
          bulk_load_hint(tc::smem_u32(ring + slot * kStageBytes), a.delta + row * a.ld + c0, bytes,
                         tc::smem_u32(&full[slot]), pol);
        }
      }
    }
  } else if (warp < 2 + kGroup / 32) {
    // ------------------------------------------------------------ norm consumers
    // squares of every client (fp64), the CTA partial -> partial[k, b], counter[k]++.  They never
    // wait on other CTAs, only stay at most one client ahead of this CTA's accumulate group
    // (so at most two clients' rows need to live in L2).
    const int gt = threadIdx.x - 64, gw = gt >> 5;
    const int64_t colA = slice_lo + 4 * gt, colB = colA + 4 * kGroup;  // this thread's two float4 per row
    int ni = 0;
    for (int k = 0; k < a.C; ++k) {
      if (k > a.lead) {
        const long long t0 = clock64();
        while (ld_acquire_cta(&acc_done) < k - a.lead) {
          __nanosleep(32);
          if (clock64() - t0 > kSpinLimit) __trap();  // a lost peer must fail loudly, never hang
        }
      }
      double ss0 = 0.0, ss1 = 0.0;
      for (int s = 0; s < nst; ++s, ++ni) {
        const int j0 = s * kRowsPerStage;
        const int slot = ni % kNormStages;
        mbar_wait_spin(&norm_full[slot], (ni / kNormStages) & 1);
        const float4* st = reinterpret_cast<const float4*>(norm_ring + slot * kStageBytes);
#pragma unroll
        for (int r = 0; r < kRowsPerStage; ++r) {
          if (j0 + r < nr) {
            const int64_t ro = (int64_t)(j0 + r) * kRowF;
            ss0 += sq4(mask_tail(st[r * (kRowF / 4) + gt], colA + ro, a.D));
            ss1 += sq4(mask_tail(st[r * (kRowF / 4) + kGroup + gt], colB + ro, a.D));
          }
        }
#ifdef FB_RING_PROXY_FENCE
        tc::fence_proxy_async();  // (generic reads of the slot ordered before the next bulk write)
#endif
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&norm_empty[slot]);
      }
      const double sw = warp_sum(ss0 + ss1);
      if (lane == 0) red[k & 1][gw] = sw;
      bar_group(1);
      if (gt == 0) {
        double tot = 0.0;
#pragma unroll
        for (int i = 0; i < kGroup / 32; ++i) tot += red[k & 1][i];
        a.partial[(int64_t)k * G + b] = tot;
        red_release_add(a.counter + k, 1u);  // (release: the partial is visible first)
      }
    }
  } else {
    // -------------------------------------------------------- accumulate consumers
    // coef[k] * client k, re-read from L2, into the TMEM / shared-memory accumulators
    const int gt = threadIdx.x - 64 - kGroup, gw = gt >> 5;
    // TMEM: a warp may touch lanes 32 * (warp % 4) .. + 31; the 2 warps sharing a lane quarter
    // take disjoint 256-column halves -> 32 slice rows x two float4 per thread
    const uint32_t tacc = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(256 * (gw >> 2));
    const int64_t colA = slice_lo + 4 * gt, colB = colA + 4 * kGroup;
    float zero32[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) zero32[i] = 0.f;
    for (int j = 0; j < kTmemRows; j += 4) tmem_st32f(tacc + 8 * j, zero32);
    for (int j = kTmemRows; j < nr; ++j) {
      sacc[(j - kTmemRows) * (kRowF / 4) + gt] = make_float4(0.f, 0.f, 0.f, 0.f);
      sacc[(j - kTmemRows) * (kRowF / 4) + kGroup + gt] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    tmem_st_wait();
    // TMEM column layout per thread and 4-row stage: [row r: A.xyzw (4 cols), B.xyzw (4 cols)]
    auto flush_or_emit = [&](bool emit, bool first) {
      for (int j0 = 0; j0 < nr; j0 += 4) {
        float v[32];
        if (j0 < kTmemRows) {
          tmem_ld32f(tacc + 8 * j0, v);
          if (!emit) tmem_st32f(tacc + 8 * j0, zero32);
        } else {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            float4 x = make_float4(0.f, 0.f, 0.f, 0.f), y = x;
            if (j0 + r < nr) {
              float4& sx = sacc[(j0 + r - kTmemRows) * (kRowF / 4) + gt];
              float4& sy = sacc[(j0 + r - kTmemRows) * (kRowF / 4) + kGroup + gt];
              x = sx;
              y = sy;
              if (!emit) sx = sy = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            v[8 * r + 0] = x.x; v[8 * r + 1] = x.y; v[8 * r + 2] = x.z; v[8 * r + 3] = x.w;
            v[8 * r + 4] = y.x; v[8 * r + 5] = y.y; v[8 * r + 6] = y.z; v[8 * r + 7] = y.w;
          }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t col = (h ? colB : colA) + (int64_t)(j0 + r) * kRowF;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (j0 + r < nr && col + q < a.D) {
                const double x = (double)v[8 * r + 4 * h + q];
                if (emit) {
                  double sum = x;
                  if (a.C > kFlush) sum += a.agg64[col + q];
                  if (a.accumulate) sum += (double)a.agg[col + q];
                  a.agg[col + q] = (float)sum;
                } else {
                  a.agg64[col + q] = (first ? 0.0 : a.agg64[col + q]) + x;
                }
              }
            }
          }
        }
      }
      tmem_st_wait();
    };
    int ai = 0;
    for (int k = 0; k < a.C; ++k) {
      // coef[k]: wait until every CTA published its partial of client k, sum the G partials
      // in a fixed order (the same bits in every CTA)
      // coef[k]: wait until every CTA published its partial of client k, sum the G partials
      // in a fixed order (the same bits in every CTA)
      if (gw == 0) {
        if (lane == 0) {
          const long long t0 = clock64();
          while (ld_relaxed(a.counter + k) < (unsigned)G) {
            __nanosleep(32);
            if (clock64() - t0 > kSpinLimit) __trap();  // a lost peer must fail loudly, never hang
          }
          fence_acq_rel();
        }
        __syncwarp();
        double p = 0.0;
        for (int i = lane; i < G; i += 32) p += __ldcg(a.partial + (int64_t)k * G + i);
        p = warp_sum(p);
        if (lane == 0) {
          const double wc = (double)__ldg(a.w + k);
          const double nrm = fabs(wc) * sqrt(p);
          const bool bad = !isfinite(nrm);
          const bool clip = !bad && a.bound > 0.0 && nrm > a.bound;
          const float c = bad ? 0.0f : (float)(clip ? wc * (a.bound / nrm) : wc);
          s_cf = c;
          if (b == 0) {
            a.norm[k] = nrm;
            a.clipped[k] = clip;
            a.nonfinite[k] = bad;
            a.coef[k] = c;
          }
        }
      }
      bar_group(2);
      const float cf = s_cf;
      for (int s = 0; s < nst; ++s, ++ai) {
        const int j0 = s * kRowsPerStage;
        const int slot = ai % kAccStages;
        mbar_wait_spin(&acc_full[slot], (ai / kAccStages) & 1);
        const float4* st = reinterpret_cast<const float4*>(acc_ring + slot * kStageBytes);
        if (j0 < kTmemRows) {
          float acc[32];
          tmem_ld32f(tacc + 8 * j0, acc);
#pragma unroll
          for (int r = 0; r < kRowsPerStage; ++r) {
            const float4 x = st[r * (kRowF / 4) + gt], y = st[r * (kRowF / 4) + kGroup + gt];
            acc[8 * r + 0] = fmaf(cf, x.x, acc[8 * r + 0]);
            acc[8 * r + 1] = fmaf(cf, x.y, acc[8 * r + 1]);
            acc[8 * r + 2] = fmaf(cf, x.z, acc[8 * r + 2]);
            acc[8 * r + 3] = fmaf(cf, x.w, acc[8 * r + 3]);
            acc[8 * r + 4] = fmaf(cf, y.x, acc[8 * r + 4]);
            acc[8 * r + 5] = fmaf(cf, y.y, acc[8 * r + 5]);
            acc[8 * r + 6] = fmaf(cf, y.z, acc[8 * r + 6]);
            acc[8 * r + 7] = fmaf(cf, y.w, acc[8 * r + 7]);
          }
          tmem_st32f(tacc + 8 * j0, acc);
        } else {
#pragma unroll
          for (int r = 0; r < kRowsPerStage; ++r) {
            if (j0 + r < nr) {
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const float4 u = st[r * (kRowF / 4) + h * kGroup + gt];
                float4& v = sacc[(j0 + r - kTmemRows) * (kRowF / 4) + h * kGroup + gt];
                v.x = fmaf(cf, u.x, v.x);
                v.y = fmaf(cf, u.y, v.y);
                v.z = fmaf(cf, u.z, v.z);
                v.w = fmaf(cf, u.w, v.w);
              }
            }
          }
        }
#ifdef FB_RING_PROXY_FENCE
        tc::fence_proxy_async();
#endif
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&acc_empty[slot]);
      }
      tmem_st_wait();  // this client's accumulator stores land before the next client reads them
      // clients 0..k accumulated: flush a full fp32 block into the fp64 accumulator
      if (((k + 1) % kFlush) == 0 && k + 1 < a.C) flush_or_emit(false, k + 1 == kFlush);
      bar_group(2);  // (all of this group is done with client k and with s_cf)
      if (gt == 0) st_release_cta(&acc_done, k + 1);
    }
    // epilogue: agg (+)= fp64 block sum + the open fp32 block
    flush_or_emit(true, false);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 0) tc::tmem_dealloc<512>(tmem_base);
}

int g_sms = 0;
int sms() {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}

int64_t max_columns() { return (int64_t)sms() * kMaxRows * kRowF; }

size_t align256(size_t n) { return (n + 255) & ~size_t(255); }

int64_t workspace_bytes(int C, int64_t D) {
  const int G = sms();
  size_t n = align256(sizeof(double) * (size_t)C * G) + align256(sizeof(unsigned) * (size_t)C);
  if (C > kFlush) n += align256(sizeof(double) * (size_t)D);
  return (int64_t)n;
}

}  // namespace
}  // namespace fb

extern "C" {

int64_t fb_clip_aggregate_max_columns(void) { return fb::max_columns(); }

int64_t fb_clip_aggregate_workspace_bytes(int num_clients, int64_t D) {
  if (num_clients < 0 || D < 0) return 0;
  return fb::workspace_bytes(num_clients, D);
}

static int clip_aggregate(const float* delta, const int32_t* rows, int64_t ld_delta, int num_clients, int64_t D, const float* w,
                          double bound, double* norm, float* coef, int32_t* clipped, int32_t* nonfinite,
                          float* agg, int accumulate, void* workspace, int64_t workspace_bytes, void* stream) {
  FB_REQUIRE(num_clients >= 0 && D >= 0 && ld_delta >= D, "clip_aggregate: bad shape (C=%d D=%lld ld=%lld)",
             num_clients, (long long)D, (long long)ld_delta);
  FB_UNSUPPORTED(D <= fb::max_columns(), "clip_aggregate: D=%lld exceeds the on-chip slice capacity %lld",
                 (long long)D, (long long)fb::max_columns());
  FB_UNSUPPORTED((ld_delta & 3) == 0 && (reinterpret_cast<uintptr_t>(delta) & 15) == 0,
                 "clip_aggregate: rows must be 16-byte aligned (ld %% 4 == 0)");
  cudaStream_t s = fb::as_stream(stream);
  if (D == 0) return FB_OK;
  if (num_clients == 0) {
    if (!accumulate) cudaMemsetAsync(agg, 0, sizeof(float) * D, s);
    return fb::launch_status("clip_aggregate(empty)");
  }
  FB_REQUIRE(workspace_bytes >= fb::workspace_bytes(num_clients, D), "clip_aggregate: workspace %lld bytes too small",
             (long long)workspace_bytes);
  const int G = fb::sms();
  char* ws = static_cast<char*>(workspace);
  fb::Args a;
  a.delta = delta;
  a.rows = rows;
  a.ld = ld_delta;
  a.C = num_clients;
  a.D = D;
  a.w = w;
  a.bound = bound;
  a.norm = norm;
  a.coef = coef;
  a.clipped = clipped;
  a.nonfinite = nonfinite;
  a.agg = agg;
  a.accumulate = accumulate;
  a.partial = reinterpret_cast<double*>(ws);
  ws += fb::align256(sizeof(double) * (size_t)num_clients * G);
  a.counter = reinterpret_cast<unsigned*>(ws);
  ws += fb::align256(sizeof(unsigned) * (size_t)num_clients);
  a.agg64 = num_clients > fb::kFlush ? reinterpret_cast<double*>(ws) : nullptr;
  // the norm group may run 2 clients ahead of the accumulate group when 3 clients' rows fit
  // well inside L2 (measured: D = 4 M 0.52 -> 0.58 of the roofline); at 10 M one client ahead
  a.lead = 12.0 * (double)ld_delta <= 64e6 ? 2 : 1;
  cudaMemsetAsync(a.counter, 0, sizeof(unsigned) * (size_t)num_clients, s);
  void* args[] = {&a};
  cudaError_t e = cudaSuccess;
  // ring depths: 3 x 32 KB from HBM, 3 x 32 KB re-read from L2 (measured best of 3/3, 4/2, 2/4)
  auto kfn = fb::clip_aggregate_fused_kernel<3, 3>;
  constexpr size_t smem = fb::smem_bytes<3, 3>();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  FB_LAUNCH("clip_aggregate_fused_kernel", s,
            e = cudaLaunchCooperativeKernel((const void*)kfn, dim3(G), dim3(fb::kT), args, smem, s));
  if (e != cudaSuccess) {
    fb::set_error("clip_aggregate: cooperative launch failed: %s", cudaGetErrorString(e));
    return FB_ERR_CUDA;
  }
  return fb::launch_status("clip_aggregate_fused_kernel");
}

int fb_clip_aggregate_f32(const float* delta, int64_t ld_delta, int num_clients, int64_t D, const float* w,
                          double bound, double* norm, float* coef, int32_t* clipped, int32_t* nonfinite,
                          float* agg, int accumulate, void* workspace, int64_t workspace_bytes, void* stream) {
  return clip_aggregate(delta, nullptr, ld_delta, num_clients, D, w, bound, norm, coef, clipped, nonfinite, agg,
                        accumulate, workspace, workspace_bytes, stream);
}

int fb_clip_aggregate_rows_f32(const float* delta, const int32_t* rows, int64_t ld_delta, int num_clients, int64_t D,
                               const float* w, double bound, double* norm, float* coef, int32_t* clipped,
                               int32_t* nonfinite, float* agg, int accumulate, void* workspace,
                               int64_t workspace_bytes, void* stream) {
  FB_REQUIRE(rows != nullptr || num_clients == 0, "clip_aggregate_rows: null rows");
  return clip_aggregate(delta, rows, ld_delta, num_clients, D, w, bound, norm, coef, clipped, nonfinite, agg,
                        accumulate, workspace, workspace_bytes, stream);
}

}  // extern "C"
