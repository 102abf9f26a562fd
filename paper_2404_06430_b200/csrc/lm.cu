// Config C: the StackOverflow-shaped transformer language model
// (models.TransformerLM), local SGD
// of a whole cohort at once and the pre-training evaluation.
//
// The reference has no LM: the arithmetic is the oracle's TransformerLM
// (oracle/port.py, pinned to float64 autograd), trained through the
// reference's generic update rule (fedsim/models/models.py:53-79):
//   theta <- theta - lr * (grad + prox_mu * (theta - theta_t) + control),
// batches in perms order, the tail batch kept, the batch loss the mean
// cross-entropy over the batch's non-pad targets.
//
// Layout.  A wave of W clients is trained together, every client's step-s
// minibatch (B sentences x L positions = T rows) side by side: activations are
// [W, T, width] fp32, each client's weights a row of Wc [W, D] (its current
// theta) and its gradient a row of G [W, D], in TransformerLM.param_dims
// order (PyTorch [out, in] weight layouts).  One step is ~45 launches over the
// wave: a grouped (per-client) tiled GEMM for every projection -- forward
// Y = X W^T (NT), backward dX = dY W (NN) and dW = dY^T X (TN) -- plus
// attention (one warp per sentence x head, L <= 32), residual + LayerNorm
// (one warp per row), the vocabulary softmax-CE (one CTA per row), bias /
// gain column sums in a fixed row order, the deterministic embedding
// scatter, and the SGD step.  Every reduction has a fixed order, so reruns
// are bit-identical.
//
// Evaluation runs the same forward with the shared theta (weight stride 0)
// over the cohort's sentences in chunks and sums per-sentence loss / hits
// into each client's totals in sentence order.

#include <math.h>
#include <stdint.h>

#include <vector>

#include "fb_common.cuh"
#include "grouped_gemm.cuh"
#include "tc_common.cuh"

#include <cudaTypedefs.h>

namespace fb {
namespace lm {

struct Dims {
  int V, d, H, dh, F, layers, L;
};

// entry offsets inside one layer (models.TransformerLM.param_dims order)
struct LayerOff {
  int64_t in_w, in_b, out_w, out_b, l1_w, l1_b, l2_w, l2_b, n1_w, n1_b, n2_w, n2_b, size;
};

inline LayerOff layer_off(const Dims& m) {
  LayerOff o;
  const int64_t d = m.d, F = m.F;
  o.in_w = 0;
  o.in_b = o.in_w + 3 * d * d;
  o.out_w = o.in_b + 3 * d;
  o.out_b = o.out_w + d * d;
  o.l1_w = o.out_b + d;
  o.l1_b = o.l1_w + F * d;
  o.l2_w = o.l1_b + F;
  o.l2_b = o.l2_w + d * F;
  o.n1_w = o.l2_b + d;
  o.n1_b = o.n1_w + d;
  o.n2_w = o.n1_b + d;
  o.n2_b = o.n2_w + d;
  o.size = o.n2_b + d;
  return o;
}
inline int64_t num_params(const Dims& m) { return (int64_t)m.V * m.d + (int64_t)m.layers * layer_off(m).size; }
inline int64_t layer_base(const Dims& m, int l) { return (int64_t)m.V * m.d + (int64_t)l * layer_off(m).size; }

// ------------------------------------------------------------------ GEMM
// (struct Gemm: grouped_gemm.cuh)
constexpr int BM = 64, BN = 64, BK = 16, GT = 256;

template <bool TA, bool TB>
__global__ void __launch_bounds__(GT) gemm_kernel(const Gemm g) {
  const int z = blockIdx.z;
  if (g.active && !g.active[z]) return;
  __shared__ float As[2][BK][BM + 4];
  __shared__ float Bs[2][BK][BN + 4];
  const float* A = g.A + (int64_t)z * g.sA;
  const float* B = g.B + (int64_t)z * g.sB;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  float ra[4], rb[4];
  // element i of this thread's share of a tile: (row-of-16, k) for NT-style loads, (k, col) otherwise
  auto load_a = [&](int k0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = tid + i * GT;
      int m, k;
      if (TA) { k = idx / BM; m = idx % BM; } else { m = idx / BK; k = idx % BK; }
      const int gm = m0 + m, gk = k0 + k;
      float v = 0.f;
      if (gm < g.M && gk < g.K) v = TA ? A[(int64_t)gk * g.lda + gm] : A[(int64_t)gm * g.lda + gk];
      ra[i] = g.relu_a ? fmaxf(v, 0.f) : v;
    }
  };
  auto load_b = [&](int k0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = tid + i * GT;
      int n, k;
      if (TB) { n = idx / BK; k = idx % BK; } else { k = idx / BN; n = idx % BN; }
      const int gn = n0 + n, gk = k0 + k;
      float v = 0.f;
      if (gn < g.N && gk < g.K) v = TB ? B[(int64_t)gn * g.ldb + gk] : B[(int64_t)gk * g.ldb + gn];
      rb[i] = g.relu_b ? fmaxf(v, 0.f) : v;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = tid + i * GT;
      if (TA) As[buf][idx / BM][idx % BM] = ra[i]; else As[buf][idx % BK][idx / BK] = ra[i];
      if (TB) Bs[buf][idx % BK][idx / BK] = rb[i]; else Bs[buf][idx / BN][idx % BN] = rb[i];
    }
  };
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  const int nk = (g.K + BK - 1) / BK;
  load_a(0);
  load_b(0);
  store(0);
  __syncthreads();
  for (int t = 0; t < nk; ++t) {
    const int cur = t & 1;
    if (t + 1 < nk) {  // next tile's global loads in flight during this tile's math
      load_a((t + 1) * BK);
      load_b((t + 1) * BK);
    }
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&As[cur][kk][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[cur][kk][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (t + 1 < nk) store(cur ^ 1);
    __syncthreads();
  }
  float* C = g.C + (int64_t)z * g.sC;
  const float* bias = g.bias ? g.bias + (int64_t)z * g.sBias : nullptr;
  const float* aux = g.aux ? g.aux + (int64_t)z * g.sAux : nullptr;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= g.N) continue;
      float v = g.alpha * acc[i][j];
      float* c = C + (int64_t)m * g.ldc + n;
      if (g.beta != 0.f) v = fmaf(g.beta, *c, v);
      if (bias) v += bias[n];
      if (aux && !(aux[(int64_t)m * g.ldaux + n] > 0.f)) v = 0.f;
      *c = v;
    }
  }
}

// 128 x 128 tiles, 8 x 8 outputs per thread (two 4 x 4 blocks 64 apart in each
// dimension), BK = 8, double-buffered shared memory: 4 LDS.128 feed 64 FFMA, so the
// FMA pipe, not shared-memory bandwidth, bounds it (the 64 x 64 / 4 x 4 kernel above
// spends 2 LDS.128 per 16 FFMA).  kVec: 128-bit global loads along the contiguous
// dimension (every row 16-byte aligned, extent % 4 == 0); else scalar.
constexpr int BM2 = 128, BN2 = 128, BK2 = 8;

template <bool TA, bool TB, bool kVec>
__global__ void __launch_bounds__(GT) gemm_big_kernel(const Gemm g) {
  const int z = blockIdx.z;
  if (g.active && !g.active[z]) return;
  __shared__ __align__(16) float As[2][BK2][BM2];
  __shared__ __align__(16) float Bs[2][BK2][BN2];
  const float* A = g.A + (int64_t)z * g.sA;
  const float* B = g.B + (int64_t)z * g.sB;
  const int m0 = blockIdx.y * BM2, n0 = blockIdx.x * BN2;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  float4 ra, rb;
  // each thread moves 4 consecutive elements along the contiguous dimension of A and of B
  auto fetch4 = [&](const float* base, int64_t ld, bool trans, int rows, int kdim, int r0, int k0, bool relu) {
    // trans: element (r, k) at base[k * ld + r] (r contiguous); else base[r * ld + k] (k contiguous)
    int r, k;
    if (trans) { k = tid >> 5; r = (tid & 31) * 4; } else { r = tid >> 1; k = (tid & 1) * 4; }
    const int gr = r0 + r, gk = k0 + k;
    float v[4];
    if (kVec) {
      if (trans) {
        if (gk < kdim && gr < rows) {
          const float4 x = *reinterpret_cast<const float4*>(base + (int64_t)gk * ld + gr);
          v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
        } else {
          v[0] = v[1] = v[2] = v[3] = 0.f;
        }
      } else {
        if (gr < rows && gk < kdim) {
          const float4 x = *reinterpret_cast<const float4*>(base + (int64_t)gr * ld + gk);
          v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
        } else {
          v[0] = v[1] = v[2] = v[3] = 0.f;
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int rr = trans ? gr + q : gr, kk = trans ? gk : gk + q;
        v[q] = (rr < rows && kk < kdim) ? (trans ? base[(int64_t)kk * ld + rr] : base[(int64_t)rr * ld + kk]) : 0.f;
      }
    }
    if (relu) {
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = fmaxf(v[q], 0.f);
    }
    return make_float4(v[0], v[1], v[2], v[3]);
  };
  auto store = [&](int buf) {
    // A: As[k][m]; B: Bs[k][n]
    if (TA) {
      *reinterpret_cast<float4*>(&As[buf][tid >> 5][(tid & 31) * 4]) = ra;
    } else {
      const int r = tid >> 1, k = (tid & 1) * 4;
      As[buf][k + 0][r] = ra.x; As[buf][k + 1][r] = ra.y; As[buf][k + 2][r] = ra.z; As[buf][k + 3][r] = ra.w;
    }
    if (!TB) {
      *reinterpret_cast<float4*>(&Bs[buf][tid >> 5][(tid & 31) * 4]) = rb;
    } else {
      const int r = tid >> 1, k = (tid & 1) * 4;
      Bs[buf][k + 0][r] = rb.x; Bs[buf][k + 1][r] = rb.y; Bs[buf][k + 2][r] = rb.z; Bs[buf][k + 3][r] = rb.w;
    }
  };
  auto fetch = [&](int k0) {
    ra = fetch4(A, g.lda, TA, g.M, g.K, m0, k0, g.relu_a);
    rb = fetch4(B, g.ldb, !TB, g.N, g.K, n0, k0, g.relu_b);
  };
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  const int nk = (g.K + BK2 - 1) / BK2;
  fetch(0);
  store(0);
  __syncthreads();
  for (int t = 0; t < nk; ++t) {
    const int cur = t & 1;
    if (t + 1 < nk) fetch((t + 1) * BK2);
#pragma unroll
    for (int kk = 0; kk < BK2; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[cur][kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[cur][kk][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[cur][kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[cur][kk][64 + tx * 4]);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (t + 1 < nk) store(cur ^ 1);
    __syncthreads();
  }
  float* C = g.C + (int64_t)z * g.sC;
  const float* bias = g.bias ? g.bias + (int64_t)z * g.sBias : nullptr;
  const float* aux = g.aux ? g.aux + (int64_t)z * g.sAux : nullptr;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (n >= g.N) continue;
      float v = g.alpha * acc[i][j];
      float* c = C + (int64_t)m * g.ldc + n;
      if (g.beta != 0.f) v = fmaf(g.beta, *c, v);
      if (bias) v += bias[n];
      if (aux && !(aux[(int64_t)m * g.ldaux + n] > 0.f)) v = 0.f;
      *c = v;
    }
  }
}

// ------------------------------------------------------- tcgen05 3xTF32 GEMM
// The same grouped C = op(A) op(B) on the 5th-gen tensor cores.  kind::tf32 reads
// K-major operands only, and an fp32-accurate product needs the 3xTF32 split
// (hi*hi + hi*lo + lo*hi, hi = rna_tf32(x), lo = rna_tf32(x - hi): ~2^-22 of the
// summands, fp32 exponent range, no scaling).  Per 32-wide K slice:
//   * a producer warp TMA-loads the raw fp32 A (128 rows) and B (BN rows) tiles
//     -- K-major operands as SWIZZLE_128B boxes {32 k, rows}, M/N-contiguous ones
//     as plain boxes {rows, 32 k} -- into a ring (3-D tensor maps, the client as
//     the outer coordinate), completion counted on an mbarrier;
//   * 4 converter warps split in shared memory: a K-major tile's hi is rounded in
//     place and its lo written at the same swizzled offset (one 16-byte chunk per
//     step); an M/N-contiguous tile is transposed into K-major SW128 hi / lo tiles;
//   * one warp issues the MMAs (M = 128, N = BN, K = 8: three per K step) into a
//     TMEM window; every 2 K slices (24 MMAs -- one long chain drifted 1.5e-4 at
//     K = 10 004) the window is handed to
//   * 4 epilogue warps that fold it into fp32 registers and finally apply alpha /
//     beta / bias / ReLU-mask with 128-bit stores.
// One output tile per CTA; grid = tiles x clients.
constexpr int TCM = 128;                 // M tile (UMMA M)
constexpr int TCK = 32;                  // K slice per stage = one 128-byte swizzle row
constexpr int TC_CONV = 8;               // converter warps (8 vs 4: TN 30 -> 27, NN 48 -> 46 ms per 2 iterations)
constexpr int TC_EPI = 8;                // epilogue warps: 2 per TMEM lane quarter, half the columns each
constexpr int TC_THREADS = 32 * (2 + TC_CONV + TC_EPI);
constexpr int TC_WIN = 2;                // K slices per TMEM window

template <bool TA, bool TB, int BNT>
struct TcCfg {
  static constexpr bool AK = !TA, BK_ = TB;          // operand already K-major in memory
  static constexpr int A_T = TCM * 128, B_T = BNT * 128;  // one K-major tile (hi or lo)
  static constexpr int A_RAW = TCM * TCK * 4, B_RAW = BNT * TCK * 4;
  // stage: [A raw (= hi when K-major)] [A hi (M-contiguous only)] [A lo] [B raw] [B hi] [B lo]
  static constexpr int A_HI = AK ? 0 : A_RAW, A_LO = AK ? A_RAW : A_RAW + A_T;
  static constexpr int B0 = A_LO + A_T;
  static constexpr int B_HI = BK_ ? B0 : B0 + B_RAW, B_LO = BK_ ? B0 + B_RAW : B0 + B_RAW + B_T;
  static constexpr int STAGE = B_LO + B_T;
  static constexpr int STAGES = STAGE <= 64 * 1024 ? 3 : 2;
  static constexpr int EPI_BYTES = TC_EPI * 32 * 33 * 4;  // per-warp 32 x 32 transpose tiles (plain stores)
  static constexpr int SMEM = 1024 + STAGES * STAGE + 256 + EPI_BYTES;
  static_assert(SMEM <= 232448, "tcgen05 GEMM shared memory");
  static constexpr uint32_t IDESC = tc::idesc_tf32(TCM, BNT);
  static constexpr uint32_t TX = A_RAW + B_RAW;
};

// 3xTF32 split with BOTH parts rounded to nearest tf32: |x - hi - lo| <= 2^-23 |x|
__device__ __forceinline__ void split_rn(float x, float& hi, float& lo) {
  hi = __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
  uint32_t l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(x - hi));
  lo = __uint_as_float(l);
}
__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts4(uint32_t a, float x, float y, float z, float w) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(x), "f"(y), "f"(z), "f"(w) : "memory");
}

// K-major raw tile of `rows` x 32 k (SW128): hi in place, lo at the same offset
__device__ __forceinline__ void conv_kmajor(uint32_t raw, uint32_t lo, int rows, bool relu, int ct) {
  constexpr int NT = 32 * TC_CONV;
  for (int i = ct; i < rows * 8; i += NT) {
    const uint32_t off = (uint32_t)i * 16;
    const float4 v = lds4(raw + off);
    const float x[4] = {v.x, v.y, v.z, v.w};
    float h[4], l[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) split_rn(relu ? fmaxf(x[q], 0.f) : x[q], h[q], l[q]);
    sts4(raw + off, h[0], h[1], h[2], h[3]);
    sts4(lo + off, l[0], l[1], l[2], l[3]);
  }
}
// M/N-contiguous raw tile [32 k][rows] -> K-major SW128 hi / lo tiles
__device__ __forceinline__ void conv_mnmajor(uint32_t raw, uint32_t hi, uint32_t lo, int rows, bool relu, int ct) {
  constexpr int NT = 32 * TC_CONV;
  for (int i = ct; i < rows * 8; i += NT) {
    const int r = i % rows, kc = (i / rows) * 4;  // consecutive threads: consecutive rows (banks)
    float h[4], l[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float x = tc::lds_f32(raw + (uint32_t)((kc + q) * rows + r) * 4);
      split_rn(relu ? fmaxf(x, 0.f) : x, h[q], l[q]);
    }
    const uint32_t off = tc::sw128_offset(r, kc);
    sts4(hi + off, h[0], h[1], h[2], h[3]);
    sts4(lo + off, l[0], l[1], l[2], l[3]);
  }
}

// Persistent: CTA b takes tiles b, b + grid, ... of the (client, m-tile, n-tile) space
// (idle clients' tiles skipped by every role alike); the stage ring and the two TMEM
// windows run on across tile boundaries, so one tile's epilogue overlaps the next
// tile's loads, conversion and MMAs.
template <bool TA, bool TB, int BNT>
__global__ void __launch_bounds__(TC_THREADS, 1) gemm_tc_kernel(const __grid_constant__ CUtensorMap ma,
                                                                const __grid_constant__ CUtensorMap mb,
                                                                const Gemm g, int a_batched, int b_batched,
                                                                int batch) {
  using Cfg = TcCfg<TA, TB, BNT>;
  constexpr int S = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* rfull = reinterpret_cast<uint64_t*>(sm + S * Cfg::STAGE);  // raw tiles landed
  uint64_t* cfull = rfull + S;                                         // split tiles ready
  uint64_t* empty = cfull + S;                                         // MMAs of the stage done
  uint64_t* tfull = empty + S;                                         // [2] window accumulated
  uint64_t* tempty = tfull + 2;                                        // [2] window drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* epi_tile = reinterpret_cast<float*>(sm + S * Cfg::STAGE + 256);  // [TC_EPI][32][33]
  // coalesced epilogue for alpha * acc (+ bias); beta / ReLU-mask epilogues keep the row-per-lane
  // path (their per-row reads serialise behind the stores in the transposed loop: LM NN
  // 23.5 -> 34.6 ms per iteration)
  const bool plain = g.beta == 0.f && !g.aux;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tn = (g.N + BNT - 1) / BNT, tm = (g.M + TCM - 1) / TCM;
  const int tiles = tn * tm * batch;
  const int nk = (g.K + TCK - 1) / TCK;
  const int nwin = (nk + TC_WIN - 1) / TC_WIN;  // windows per tile
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      tc::mbar_init(&rfull[i], 1);
      tc::mbar_init(&cfull[i], TC_CONV);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], TC_EPI);
    }
    tc::fence_mbar_init();
  }
  constexpr uint32_t kCols = 2 * BNT <= 256 ? 256 : 512;  // two accumulator windows
  if (warp == 1) tc::tmem_alloc<kCols>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t s0 = tc::smem_u32(sm);
  // tile -> (client z, m0, n0); n fastest so consecutive tiles of a CTA share the A rows
  auto geom = [&](int tile, int& z, int& m0, int& n0) -> bool {
    z = tile / (tn * tm);
    const int r = tile - z * tn * tm, mt = r / tn;
    m0 = mt * TCM;
    n0 = (r - mt * tn) * BNT;
    return !g.active || g.active[z];
  };

  if (warp == 0) {
    // -------------------------------------------------------------- producer
    if (lane == 0) {
      tc::tma_prefetch(&ma);
      tc::tma_prefetch(&mb);
      int t = 0;  // global stage counter
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        int z, m0, n0;
        if (!geom(tile, z, m0, n0)) continue;
        const int za = a_batched ? z : 0, zb = b_batched ? z : 0;
        for (int kk = 0; kk < nk; ++kk, ++t) {
          const int st = t % S;
          if (t >= S) tc::mbar_wait(&empty[st], ((t / S) - 1) & 1);
          tc::mbar_arrive_expect_tx(&rfull[st], Cfg::TX);
          uint8_t* base = sm + st * Cfg::STAGE;
          const int k0 = kk * TCK;
          if (Cfg::AK) tc::tma_load_3d(base, &ma, k0, m0, za, &rfull[st]);
          else tc::tma_load_3d(base, &ma, m0, k0, za, &rfull[st]);
          if (Cfg::BK_) tc::tma_load_3d(base + Cfg::B0, &mb, k0, n0, zb, &rfull[st]);
          else tc::tma_load_3d(base + Cfg::B0, &mb, n0, k0, zb, &rfull[st]);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    int t = 0, w = 0;  // global stage / window counters
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      int z, m0, n0;
      if (!geom(tile, z, m0, n0)) continue;
      for (int kk = 0; kk < nk; ++kk, ++t) {
        const int st = t % S, buf = w & 1;
        if (kk % TC_WIN == 0 && w >= 2) {  // this window's buffer drained (window w - 2)?
          tc::mbar_wait(&tempty[buf], ((w >> 1) - 1) & 1);
          tc::tc_fence_after();
        }
        tc::mbar_wait(&cfull[st], (t / S) & 1);
        tc::tc_fence_after();
        if (tc::elect_one()) {
          const uint32_t d = tmem + buf * BNT;
          const uint32_t base = s0 + st * Cfg::STAGE;
          const uint32_t ah = base + Cfg::A_HI, al = base + Cfg::A_LO;
          const uint32_t bh = base + Cfg::B_HI, bl = base + Cfg::B_LO;
#pragma unroll
          for (int k8 = 0; k8 < TCK / 8; ++k8) {
            const uint32_t kb = k8 * 32;  // 8 tf32 = 32 bytes along the swizzled row
            const uint32_t acc0 = (kk % TC_WIN > 0 || k8 > 0) ? 1u : 0u;
            tc::mma_tf32(d, tc::sdesc_k128(ah + kb), tc::sdesc_k128(bh + kb), Cfg::IDESC, acc0);
            tc::mma_tf32(d, tc::sdesc_k128(ah + kb), tc::sdesc_k128(bl + kb), Cfg::IDESC, 1u);
            tc::mma_tf32(d, tc::sdesc_k128(al + kb), tc::sdesc_k128(bh + kb), Cfg::IDESC, 1u);
          }
          tc::mma_commit(&empty[st]);
          if (kk % TC_WIN == TC_WIN - 1 || kk == nk - 1) tc::mma_commit(&tfull[buf]);
        }
        __syncwarp();
        if (kk % TC_WIN == TC_WIN - 1 || kk == nk - 1) ++w;
      }
    }
  } else if (warp < 2 + TC_CONV) {
    // ------------------------------------------------------------ converters
    const int ct = threadIdx.x - 64;
    int t = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      int z, m0, n0;
      if (!geom(tile, z, m0, n0)) continue;
      for (int kk = 0; kk < nk; ++kk, ++t) {
        const int st = t % S;
        tc::mbar_wait(&rfull[st], (t / S) & 1);
        const uint32_t base = s0 + st * Cfg::STAGE;
        if (Cfg::AK) conv_kmajor(base, base + Cfg::A_LO, TCM, g.relu_a, ct);
        else conv_mnmajor(base, base + Cfg::A_HI, base + Cfg::A_LO, TCM, g.relu_a, ct);
        if (Cfg::BK_) conv_kmajor(base + Cfg::B0, base + Cfg::B_LO, BNT, g.relu_b, ct);
        else conv_mnmajor(base + Cfg::B0, base + Cfg::B_HI, base + Cfg::B_LO, BNT, g.relu_b, ct);
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&cfull[st]);
      }
    }
  } else {
    // --------------------------------------------------------------- epilogue
    // warp e = warp - 6: TMEM lane quarter warp % 4, column half e / 4
    constexpr int EH = BNT / 2;
    const int q = warp & 3, half = (warp - 2 - TC_CONV) >> 2;
    int w = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      int z, m0, n0;
      if (!geom(tile, z, m0, n0)) continue;
      const int m = m0 + q * 32 + lane;
      n0 += half * EH;  // this warp's columns
      float sum[EH];
#pragma unroll
      for (int j = 0; j < EH; ++j) sum[j] = 0.f;
      for (int wi = 0; wi < nwin; ++wi, ++w) {
        const int buf = w & 1;
        tc::mbar_wait(&tfull[buf], (w >> 1) & 1);
        tc::tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < EH; c0 += 16) {
          uint32_t v[16];
          tc::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + buf * BNT + half * EH + c0, v);
          tc::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) sum[c0 + j] += __uint_as_float(v[j]);
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&tempty[buf]);
      }
      if (plain) {
        // each 32 x 32 sub-tile goes through the warp's private smem tile
        // (row-per-lane in, column-per-lane out, 33-float pitch: conflict-free both ways), so
        // every store instruction writes 128 contiguous bytes of one output row (the
        // row-per-lane float4 stores touched 32 rows each -- the dcol / logits outputs)
        float* tile = epi_tile + (warp - 2 - TC_CONV) * (32 * 33);
        const int mrow0 = m0 + q * 32;
#pragma unroll
        for (int c0 = 0; c0 < EH; c0 += 32) {
          // (EH = 48 for the 96-wide tiles: the second sub-tile is 16 columns wide)
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c0 + j < EH) tile[lane * 33 + j] = g.alpha * sum[c0 + j];
          __syncwarp();
          const int col = n0 + c0 + lane;
          const bool live = c0 + lane < EH && col < g.N;
          const float bcol = live && g.bias ? g.bias[(int64_t)z * g.sBias + col] : 0.f;
          for (int r = 0; r < 32; ++r) {
            const int mr = mrow0 + r;
            if (live && mr < g.M) g.C[(int64_t)z * g.sC + (int64_t)mr * g.ldc + col] = tile[r * 33 + lane] + bcol;
          }
          __syncwarp();
        }
      } else if (m < g.M) {
        float* crow = g.C + (int64_t)z * g.sC + (int64_t)m * g.ldc;
        const float* bias = g.bias ? g.bias + (int64_t)z * g.sBias : nullptr;
        const float* arow = g.aux ? g.aux + (int64_t)z * g.sAux + (int64_t)m * g.ldaux : nullptr;
        // row per lane: 256-bit loads / stores (whole 32-byte sectors per lane) where the row,
        // the bias and the mask rows are 32-byte aligned; same arithmetic order as the scalar path
        const auto al32 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31) == 0; };
        const bool v8 = (g.ldc & 7) == 0 && al32(crow) && (!bias || al32(bias)) &&
                        (!arow || ((g.ldaux & 7) == 0 && al32(arow)));
#pragma unroll
        for (int j0 = 0; j0 < EH; j0 += 8) {
          const int n = n0 + j0;
          float x[8];
          if (v8 && n + 7 < g.N) {
#pragma unroll
            for (int u = 0; u < 8; ++u) x[u] = g.alpha * sum[j0 + u];
            if (g.beta != 0.f) {
              float cv[8];
              tc::ldg256(crow + n, cv);
#pragma unroll
              for (int u = 0; u < 8; ++u) x[u] = fmaf(g.beta, cv[u], x[u]);
            }
            if (bias) {
              float bv[8];
              tc::ldg256(bias + n, bv);
#pragma unroll
              for (int u = 0; u < 8; ++u) x[u] += bv[u];
            }
            if (arow) {
              float av[8];
              tc::ldg256(arow + n, av);
#pragma unroll
              for (int u = 0; u < 8; ++u)
                if (!(av[u] > 0.f)) x[u] = 0.f;
            }
            tc::stg256f(crow + n, x);
          } else {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int nn = n + u;
              if (nn < g.N) {
                float val = g.alpha * sum[j0 + u];
                if (g.beta != 0.f) val = fmaf(g.beta, crow[nn], val);
                if (bias) val += bias[nn];
                if (arow && !(arow[nn] > 0.f)) val = 0.f;
                crow[nn] = val;
              }
            }
          }
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc<kCols>(tmem);
}

// ------------------------------------------------------------ batch gather
// Client c's step-s minibatch: epoch e = s / nb, batch j = s % nb (nb = ceil(n / B)),
// sentences perms[c][e * n + j * B + i]; slots past the batch are all-pad.
// nvalid[c] = non-pad targets in the batch (0: client idle this step).
__global__ void gather_batch_kernel(const float* __restrict__ X, const int64_t* __restrict__ row_start,
                                    const int32_t* __restrict__ num_rows, const int32_t* __restrict__ perms,
                                    const int64_t* __restrict__ perm_off, int c0, int epochs, int B, int L, int step,
                                    int32_t* __restrict__ tok, int32_t* __restrict__ nvalid) {
  const int w = blockIdx.x, c = c0 + w;
  const int n = num_rows[c];
  const int nb = n > 0 ? (n + B - 1) / B : 0;
  const bool live = nb > 0 && step < epochs * nb;
  const int e = live ? step / nb : 0, j = live ? step % nb : 0;
  const int cnt = live ? min(B, n - j * B) : 0;
  int32_t* t = tok + (int64_t)w * B * (L + 1);
  __shared__ int nv;
  if (threadIdx.x == 0) nv = 0;
  __syncthreads();
  int mine = 0;
  for (int q = threadIdx.x; q < B * (L + 1); q += blockDim.x) {
    const int i = q / (L + 1), p = q - i * (L + 1);
    int v = 0;
    if (i < cnt) {
      const int r = perms[perm_off[c] + (int64_t)e * n + j * B + i];
      v = (int)X[(row_start[c] + r) * (int64_t)(L + 1) + p];
    }
    t[q] = v;
    mine += (p > 0 && v != 0);
  }
  atomicAdd(&nv, mine);  // integer: order-free
  __syncthreads();
  if (threadIdx.x == 0) nvalid[w] = nv;
}

// eval chunk: sentences [g0, g0 + cnt) of the cohort in client-major order
// (perms != nullptr: client c's evaluated sentences are epoch 0's perms[perm_off[c] + skip_c ..],
//  skip_c = min(skip, n_c): the first local step evaluates the first batch)
__global__ void gather_eval_kernel(const float* __restrict__ X, const int64_t* __restrict__ row_start,
                                   const int64_t* __restrict__ sent_off, int C, int64_t g0, int cnt, int L,
                                   int32_t* __restrict__ tok, const int32_t* __restrict__ perms,
                                   const int64_t* __restrict__ perm_off, const int32_t* __restrict__ num_rows,
                                   int skip) {
  const int i = blockIdx.x;  // sentence slot
  int32_t* t = tok + (int64_t)i * (L + 1);
  if (i >= cnt) {
    for (int p = threadIdx.x; p <= L; p += blockDim.x) t[p] = 0;
    return;
  }
  const int64_t g = g0 + i;
  int lo = 0, hi = C - 1;  // last client with sent_off <= g
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (sent_off[mid] <= g) lo = mid; else hi = mid - 1;
  }
  const int64_t j = g - sent_off[lo];
  const int64_t row = row_start[lo] + (perms ? perms[perm_off[lo] + min(skip, num_rows[lo]) + j] : j);
  for (int p = threadIdx.x; p <= L; p += blockDim.x) t[p] = (int)X[row * (L + 1) + p];
}

__global__ void positions_kernel(float* __restrict__ pe, int L, int d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L * d) return;
  const int pos = i / d, j = i - pos * d;
  const double div = exp((double)(j & ~1) * (-log(10000.0) / d));
  pe[i] = (float)((j & 1) ? cos(pos * div) : sin(pos * div));
}

// x[w, s*L + p, :] = E_w[tok[w, s, p]] * sqrt(d) + pe[p]
__global__ void embed_kernel(const int32_t* __restrict__ tok, const float* __restrict__ Wc, int64_t sW,
                             const float* __restrict__ pe, int B, int L, int d, const int32_t* __restrict__ active,
                             float* __restrict__ x) {
  const int w = blockIdx.y;
  if (active && !active[w]) return;
  const int row = blockIdx.x;  // s * L + p
  const int s = row / L, p = row - s * L;
  const int id = tok[((int64_t)w * B + s) * (L + 1) + p];
  const float* E = Wc + (int64_t)w * sW + (int64_t)id * d;
  const float sc = sqrtf((float)d);
  float* out = x + ((int64_t)w * B * L + row) * d;
  for (int j = threadIdx.x; j < d; j += blockDim.x) out[j] = fmaf(E[j], sc, pe[p * d + j]);
}

// dE_w[tok] += dx0 * sqrt(d), tokens in row order (deterministic)
__global__ void embed_bwd_kernel(const int32_t* __restrict__ tok, const float* __restrict__ dx, int B, int L, int d,
                                 const int32_t* __restrict__ active, float* __restrict__ G, int64_t sG) {
  const int w = blockIdx.x;
  if (!active[w]) return;
  const float sc = sqrtf((float)d);
  float* gE = G + (int64_t)w * sG;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    for (int r = 0; r < B * L; ++r) {
      const int s = r / L, p = r - s * L;
      const int id = tok[((int64_t)w * B + s) * (L + 1) + p];
      gE[(int64_t)id * d + j] = fmaf(dx[((int64_t)w * B * L + r) * d + j], sc, gE[(int64_t)id * d + j]);
    }
  }
}

// ----------------------------------------------------------------- attention
// one CTA per (client, sentence), one warp per head, lane i = query position i
// (L <= 32, dh <= 32, H <= 16): the sentence's [L, 3d] qkv block is staged in shared
// memory with coalesced loads (row stride 3d + 1: conflict-free per-lane rows); the
// per-row score / probability vectors live in registers (fully unrolled over 32
// positions, predicated by the causal bound)
__device__ __forceinline__ void stage_rows(float* dst, int ldd, const float* src, int64_t lds, int rows, int cols) {
  for (int e = threadIdx.x; e < rows * cols; e += blockDim.x) {
    const int r = e / cols, c = e - r * cols;
    dst[r * ldd + c] = src[(int64_t)r * lds + c];
  }
}

__global__ void __launch_bounds__(512) attn_fwd_kernel(const float* __restrict__ qkv, int B, int L, int H, int dh,
                                                       const int32_t* __restrict__ active, float* __restrict__ P,
                                                       float* __restrict__ o) {
  extern __shared__ float sh[];  // [L][3d + 1]
  const int w = blockIdx.y, s = blockIdx.x;
  if (!active[w]) return;
  const int d = H * dh, ld = 3 * d + 1;
  stage_rows(sh, ld, qkv + ((int64_t)w * B * L + (int64_t)s * L) * 3 * d, 3 * d, L, 3 * d);
  __syncthreads();
  const int h = threadIdx.x >> 5, i = threadIdx.x & 31;
  if (h >= H || i >= L) return;
  const float* q = sh + i * ld + h * dh;
  const float sc = 1.0f / sqrtf((float)dh);
  float sv[32];
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    sv[j] = -INFINITY;
    if (j <= i) {
      const float* kj = sh + j * ld + d + h * dh;
      float a = 0.f;
      for (int c = 0; c < dh; ++c) a = fmaf(q[c], kj[c], a);
      sv[j] = a * sc;
      mx = fmaxf(mx, sv[j]);
    }
  }
  float sum = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    sv[j] = j <= i ? expf(sv[j] - mx) : 0.f;
    sum += sv[j];
  }
  const float inv = 1.0f / sum;
  float* prow = P + ((((int64_t)w * B + s) * H + h) * L + i) * L;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    sv[j] *= inv;
    if (j < L) prow[j] = sv[j];
  }
  float* orow = o + ((int64_t)w * B * L + (int64_t)s * L + i) * d + h * dh;
  for (int c = 0; c < dh; ++c) {
    float a = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j <= i) a = fmaf(sv[j], sh[j * ld + 2 * d + h * dh + c], a);
    orow[c] = a;
  }
}

__global__ void __launch_bounds__(512) attn_bwd_kernel(const float* __restrict__ qkv, const float* __restrict__ P,
                                                       const float* __restrict__ dout, int B, int L, int H, int dh,
                                                       const int32_t* __restrict__ active, float* __restrict__ dqkv) {
  extern __shared__ float sh[];  // qkv [L][3d + 1] | dO [L][d + 1] | dS [H][L][33]
  const int w = blockIdx.y, s = blockIdx.x;
  if (!active[w]) return;
  const int d = H * dh, ld = 3 * d + 1, ldo = d + 1;
  float* dO = sh + L * ld;
  float* dSall = dO + L * ldo;
  const int64_t row0 = (int64_t)w * B * L + (int64_t)s * L;
  stage_rows(sh, ld, qkv + row0 * 3 * d, 3 * d, L, 3 * d);
  stage_rows(dO, ldo, dout + row0 * d, d, L, d);
  __syncthreads();
  const int h = threadIdx.x >> 5, i = threadIdx.x & 31;
  if (h >= H) return;
  float* dS = dSall + h * L * 33;
  const float* pbase = P + (((int64_t)w * B + s) * H + h) * L * L;
  const float sc = 1.0f / sqrtf((float)dh);
  if (i < L) {  // row i: dS_ij = P_ij (dP_ij - sum_j P_ij dP_ij) / sqrt(dh)
    const float* doi = dO + i * ldo + h * dh;
    float dp[32], pr[32];
    float rs = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      dp[j] = 0.f;
      pr[j] = 0.f;
      if (j <= i) {
        const float* vj = sh + j * ld + 2 * d + h * dh;
        float a = 0.f;
        for (int c = 0; c < dh; ++c) a = fmaf(doi[c], vj[c], a);
        dp[j] = a;
        pr[j] = pbase[i * L + j];
        rs = fmaf(pr[j], a, rs);
      }
    }
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < L) dS[i * 33 + j] = j <= i ? pr[j] * (dp[j] - rs) * sc : 0.f;
  }
  __syncwarp();
  if (i >= L) return;
  float* dq = dqkv + (row0 + i) * 3 * d + h * dh;
  for (int c = 0; c < dh; ++c) {  // dq_i = sum_j dS_ij k_j ; dk_i = sum_r dS_ri q_r ; dv_i = sum_r P_ri dO_r
    float aq = 0.f, ak = 0.f, av = 0.f;
    for (int j = 0; j <= i; ++j) aq = fmaf(dS[i * 33 + j], sh[j * ld + d + h * dh + c], aq);
    for (int r = i; r < L; ++r) {
      ak = fmaf(dS[r * 33 + i], sh[r * ld + h * dh + c], ak);
      av = fmaf(pbase[r * L + i], dO[r * ldo + h * dh + c], av);
    }
    dq[c] = aq;
    dq[d + c] = ak;
    dq[2 * d + c] = av;
  }
}

// --------------------------------------------------------------- LayerNorm
// out = LN(a + b) * g + beta per row of d (one warp per row); keeps xh, rstd
__global__ void add_ln_kernel(const float* __restrict__ a, const float* __restrict__ b, const float* __restrict__ gw,
                              const float* __restrict__ gb, int64_t sWc, int rows, int d, float eps,
                              const int32_t* __restrict__ active, float* __restrict__ xh, float* __restrict__ rstd,
                              float* __restrict__ out) {
  const int w = blockIdx.y;
  if (!active[w]) return;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int64_t off = ((int64_t)w * rows + r) * d;
  float y[8];
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int j = lane + 32 * u;
    y[u] = j < d ? a[off + j] + b[off + j] : 0.f;
    s += y[u];
  }
  s = warp_sum(s);
  const float mean = s / d;
  float v = 0.f;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int j = lane + 32 * u;
    const float c = j < d ? y[u] - mean : 0.f;
    v = fmaf(c, c, v);
  }
  v = warp_sum(v);
  const float rs = 1.0f / sqrtf(v / d + eps);
  const float* g = gw + (int64_t)w * sWc;
  const float* be = gb + (int64_t)w * sWc;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int j = lane + 32 * u;
    if (j < d) {
      const float h = (y[u] - mean) * rs;
      if (xh) xh[off + j] = h;
      out[off + j] = fmaf(h, g[j], be[j]);
    }
  }
  if (rstd && lane == 0) rstd[(int64_t)w * rows + r] = rs;
}

// dy = rstd * (dxh - mean(dxh) - xh * mean(dxh * xh)), dxh = dout * g
__global__ void ln_bwd_kernel(const float* __restrict__ dout, const float* __restrict__ xh,
                              const float* __restrict__ rstd, const float* __restrict__ gw, int64_t sWc, int rows,
                              int d, const int32_t* __restrict__ active, float* __restrict__ dy) {
  const int w = blockIdx.y;
  if (!active[w]) return;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int64_t off = ((int64_t)w * rows + r) * d;
  const float* g = gw + (int64_t)w * sWc;
  float dh[8], hh[8];
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int j = lane + 32 * u;
    dh[u] = j < d ? dout[off + j] * g[j] : 0.f;
    hh[u] = j < d ? xh[off + j] : 0.f;
    s1 += dh[u];
    s2 = fmaf(dh[u], hh[u], s2);
  }
  s1 = warp_sum(s1) / d;
  s2 = warp_sum(s2) / d;
  const float rs = rstd[(int64_t)w * rows + r];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int j = lane + 32 * u;
    if (j < d) dy[off + j] = rs * (dh[u] - s1 - hh[u] * s2);
  }
}

// G_w[col] = sum_r in1[w, r, col] (* in2[w, r, col]): CTA = 32 columns x 8 warps, warp u
// sums rows u, u + 8, ... in order and the 8 partials are added in warp order (fixed, so
// deterministic; 8 independent load streams per column instead of one serial one)
constexpr int kCsWarps = 8;
__global__ void __launch_bounds__(32 * kCsWarps) colsum_kernel(const float* __restrict__ in1,
                                                               const float* __restrict__ in2, int rows, int cols,
                                                               const int32_t* __restrict__ active,
                                                               float* __restrict__ G, int64_t sG) {
  __shared__ float part[kCsWarps][33];
  const int w = blockIdx.y;
  if (!active[w]) return;
  const int lane = threadIdx.x & 31, u = threadIdx.x >> 5;
  const int col = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (col < cols) {
    const int64_t base = (int64_t)w * rows * cols + col;
    if (in2) {
      for (int r = u; r < rows; r += kCsWarps) s = fmaf(in1[base + (int64_t)r * cols], in2[base + (int64_t)r * cols], s);
    } else {
      for (int r = u; r < rows; r += kCsWarps) s += in1[base + (int64_t)r * cols];
    }
  }
  part[u][lane] = s;
  __syncthreads();
  if (u == 0 && col < cols) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < kCsWarps; ++i) t += part[i][lane];
    G[(int64_t)w * sG + col] = t;
  }
}

// ------------------------------------------------------------ softmax-CE
// one CTA per row of V logits; target t = tok[w, s, p + 1] (0 = pad: ignored).
// train: logits <- (softmax - onehot) / nvalid[w] (0 for pad rows).
// eval : row_loss / row_hit (first argmax) for non-pad rows, 0 else.
constexpr int kCeT = 256;

template <bool kTrain>
__global__ void __launch_bounds__(kCeT) ce_kernel(float* __restrict__ logits, const int32_t* __restrict__ tok,
                                                  int B, int L, int V, const int32_t* __restrict__ nvalid,
                                                  float* __restrict__ row_loss, int32_t* __restrict__ row_hit) {
  const int w = blockIdx.y;
  if (kTrain && nvalid[w] == 0) return;
  const int r = blockIdx.x;  // s * L + p
  const int s = r / L, p = r - s * L;
  const int tgt = tok[((int64_t)w * B + s) * (L + 1) + p + 1];
  float* z = logits + ((int64_t)w * B * L + r) * V;
  __shared__ float red[32];
  __shared__ int redi[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (tgt == 0) {
    if (kTrain) {
      for (int v = threadIdx.x; v < V; v += kCeT) z[v] = 0.f;
    }
    if (row_loss && threadIdx.x == 0) {
      row_loss[(int64_t)w * B * L + r] = 0.f;
      row_hit[(int64_t)w * B * L + r] = 0;
    }
    return;
  }
  // max (and its first index for eval)
  float mx = -INFINITY;
  int arg = 0x7fffffff;
  for (int v = threadIdx.x; v < V; v += kCeT) {
    const float x = z[v];
    if (x > mx) { mx = x; arg = v; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, mx, o);
    const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
    if (om > mx || (om == mx && oa < arg)) { mx = om; arg = oa; }
  }
  if (lane == 0) { red[wid] = mx; redi[wid] = arg; }
  __syncthreads();
  if (wid == 0) {
    mx = lane < kCeT / 32 ? red[lane] : -INFINITY;
    arg = lane < kCeT / 32 ? redi[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, mx, o);
      const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
      if (om > mx || (om == mx && oa < arg)) { mx = om; arg = oa; }
    }
    if (lane == 0) { red[0] = mx; redi[0] = arg; }
  }
  __syncthreads();
  mx = red[0];
  arg = redi[0];
  __syncthreads();
  float se = 0.f;
  for (int v = threadIdx.x; v < V; v += kCeT) se += expf(z[v] - mx);
  se = warp_sum(se);
  if (lane == 0) red[wid] = se;
  __syncthreads();
  if (wid == 0) {
    se = lane < kCeT / 32 ? red[lane] : 0.f;
    se = warp_sum(se);
    if (lane == 0) red[0] = se;
  }
  __syncthreads();
  se = red[0];
  if (kTrain) {
    if (row_loss) {  // the first local step: its logits are the theta_t evaluation of the batch
      if (threadIdx.x == 0) {
        row_loss[(int64_t)w * B * L + r] = -(z[tgt] - mx - logf(se));
        row_hit[(int64_t)w * B * L + r] = arg == tgt;
      }
      __syncthreads();  // (z[tgt] read before it is overwritten below)
    }
    const float scale = 1.0f / (float)nvalid[w];
    const float inv = 1.0f / se;
    for (int v = threadIdx.x; v < V; v += kCeT) {
      float pr = expf(z[v] - mx) * inv;
      if (v == tgt) pr -= 1.0f;
      z[v] = pr * scale;
    }
  } else if (threadIdx.x == 0) {
    row_loss[(int64_t)w * B * L + r] = -(z[tgt] - mx - logf(se));
    row_hit[(int64_t)w * B * L + r] = arg == tgt;
  }
}

// per-sentence (in position order) then per-client (in sentence order) eval sums
__global__ void eval_accum_kernel(const float* __restrict__ row_loss, const int32_t* __restrict__ row_hit,
                                  const int64_t* __restrict__ sent_off, const int32_t* __restrict__ num_rows, int C,
                                  int64_t g0, int cnt, int L, double* __restrict__ loss, int32_t* __restrict__ correct,
                                  int skip) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int64_t nc = num_rows[c] - min(skip, num_rows[c]);
  const int64_t lo = sent_off[c] > g0 ? sent_off[c] : g0;
  const int64_t hi = sent_off[c] + nc < g0 + cnt ? sent_off[c] + nc : g0 + cnt;
  double s = 0.0;
  int k = 0;
  for (int64_t g = lo; g < hi; ++g) {
    const int64_t i = g - g0;
    double sl = 0.0;
    for (int p = 0; p < L; ++p) {
      sl += (double)row_loss[i * L + p];
      k += row_hit[i * L + p];
    }
    s += sl;
  }
  if (hi > lo) {
    loss[c] += s;
    correct[c] += k;
  }
}

// the first local step's batch rows (client w of the wave: sentences s < B, in order) added
// to the client's evaluation sums the same way eval_accum_kernel adds a chunk's
__global__ void step0_eval_kernel(const float* __restrict__ row_loss, const int32_t* __restrict__ row_hit,
                                  const int32_t* __restrict__ nvalid, int W, int B, int L,
                                  double* __restrict__ loss, int32_t* __restrict__ correct) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= W || nvalid[w] == 0) return;
  double sacc = 0.0;
  int k = 0;
  for (int s = 0; s < B; ++s) {
    double sl = 0.0;
    for (int p = 0; p < L; ++p) {
      sl += (double)row_loss[((int64_t)w * B + s) * L + p];
      k += row_hit[((int64_t)w * B + s) * L + p];
    }
    sacc += sl;
  }
  loss[w] += sacc;
  correct[w] += k;
}

// -------------------------------------------------------------- SGD step
// theta <- theta - lr * (g + mu * (theta - theta_t) + control); delta accumulates the step
__global__ void sgd_kernel(float* __restrict__ Wc, const float* __restrict__ G, int64_t sW,
                           float* __restrict__ Dl, int64_t ldD, const float* __restrict__ control, int64_t ldc,
                           int64_t D, float lr, float mu, const int32_t* __restrict__ nvalid) {
  const int w = blockIdx.y;
  if (nvalid[w] == 0) return;
  float* W = Wc + (int64_t)w * sW;
  const float* g = G + (int64_t)w * sW;
  float* dl = Dl + (int64_t)w * ldD;
  const float* ct = control ? control + (int64_t)w * ldc : nullptr;
  // 16-byte path when every row is 16-byte aligned (the workspace strides are): 5 float4
  // accesses in flight per thread instead of 5 scalars; the same arithmetic per element
  const auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if ((D & 3) == 0 && a16(W) && a16(g) && a16(dl) && (!ct || a16(ct))) {
    const int64_t D4 = D >> 2;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < D4; i += (int64_t)gridDim.x * blockDim.x) {
      const float4 gv = reinterpret_cast<const float4*>(g)[i];
      float4 dv = reinterpret_cast<float4*>(dl)[i];
      float4 wv = reinterpret_cast<float4*>(W)[i];
      const float4 cv = ct ? reinterpret_cast<const float4*>(ct)[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      float sv[4] = {gv.x, gv.y, gv.z, gv.w};
      float* dp4 = &dv.x;
      float* wp4 = &wv.x;
      const float* cp4 = &cv.x;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float x = sv[e];
        if (mu != 0.f) x = fmaf(mu, -dp4[e], x);
        if (ct) x += cp4[e];
        x *= lr;
        wp4[e] -= x;
        dp4[e] += x;
      }
      reinterpret_cast<float4*>(W)[i] = wv;
      reinterpret_cast<float4*>(dl)[i] = dv;
    }
    return;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < D; i += (int64_t)gridDim.x * blockDim.x) {
    float s = g[i];
    if (mu != 0.f) s = fmaf(mu, -dl[i], s);
    if (ct) s += ct[i];
    s *= lr;
    W[i] -= s;
    dl[i] += s;
  }
}

__global__ void init_wave_kernel(const float* __restrict__ theta_t, int64_t D, float* __restrict__ Wc, int64_t sW,
                                 float* __restrict__ Dl, int64_t ldD) {
  const int w = blockIdx.y;
  float* wc = Wc + (int64_t)w * sW;
  float* dl = Dl + (int64_t)w * ldD;
  const auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if ((D & 3) == 0 && a16(theta_t) && a16(wc) && a16(dl)) {  // 16-byte path
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (D >> 2); i += (int64_t)gridDim.x * blockDim.x) {
      reinterpret_cast<float4*>(wc)[i] = reinterpret_cast<const float4*>(theta_t)[i];
      reinterpret_cast<float4*>(dl)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    return;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < D; i += (int64_t)gridDim.x * blockDim.x) {
    wc[i] = theta_t[i];
    dl[i] = 0.f;
  }
}

__global__ void nonfinite_kernel(const float* __restrict__ Dl, int64_t ldD, int64_t D, int32_t* __restrict__ bad) {
  const int w = blockIdx.x;
  const float* dl = Dl + (int64_t)w * ldD;
  int b = 0;
  int64_t i0 = 0;
  if ((reinterpret_cast<uintptr_t>(dl) & 15) == 0) {  // 16-byte loads, 4 in flight per thread
    const float4* d4 = reinterpret_cast<const float4*>(dl);
    const int64_t n4 = D >> 2, step = 4 * (int64_t)blockDim.x;
    int64_t i = threadIdx.x;
    for (; i + 3 * blockDim.x < n4; i += step) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = d4[i + u * blockDim.x];
#pragma unroll
      for (int u = 0; u < 4; ++u) b |= !isfinite(v[u].x) | !isfinite(v[u].y) | !isfinite(v[u].z) | !isfinite(v[u].w);
    }
    for (; i < n4; i += blockDim.x) {
      const float4 v = d4[i];
      b |= !isfinite(v.x) | !isfinite(v.y) | !isfinite(v.z) | !isfinite(v.w);
    }
    i0 = n4 << 2;
  }
  for (int64_t i = i0 + threadIdx.x; i < D; i += blockDim.x) b |= !isfinite(dl[i]);
  b = __syncthreads_or(b);
  if (threadIdx.x == 0) bad[w] = b;
}

__global__ void copy_kernel(const float* __restrict__ src, float* __restrict__ dst, int64_t n_per, int64_t stride,
                            const int32_t* __restrict__ active) {
  const int w = blockIdx.y;
  if (!active[w]) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_per; i += (int64_t)gridDim.x * blockDim.x)
    dst[(int64_t)w * stride + i] = src[(int64_t)w * stride + i];
}

__global__ void ones_kernel(int32_t* p, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = 1;
}

__global__ void sent_offsets_kernel(const int32_t* __restrict__ num_rows, int C, int64_t* __restrict__ off, int skip) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int64_t s = 0;
    for (int c = 0; c < C; ++c) {
      off[c] = s;
      s += num_rows[c] - min(skip, num_rows[c]);
    }
  }
}

// ------------------------------------------------------------ workspace
struct Buf {
  size_t off = 0;
  char* base = nullptr;
  template <typename T>
  T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
};

struct Layer {
  float *xin, *qkv, *P, *o, *xh1, *r1, *x1, *z, *xh2, *r2;
};

struct Work {
  int32_t *tok, *nvalid, *active, *hit;
  int64_t* sent_off;
  float *pe, *Wc, *G, *xf, *logits, *dx, *dx1, *dz, *dqkv, *dtmp, *a, *f, *rloss;
  std::vector<Layer> layer;
};

// W groups of B sentences; train = with gradient / client-weight buffers
inline Work carve(const Dims& m, int W, int B, bool train, Buf& b) {
  const int64_t T = (int64_t)B * m.L, d = m.d, D = num_params(m);
  const int64_t sW = (D + 3) & ~int64_t(3);
  Work k;
  k.tok = b.take<int32_t>((size_t)W * B * (m.L + 1));
  k.nvalid = b.take<int32_t>(W);
  k.active = b.take<int32_t>(W);
  k.sent_off = b.take<int64_t>(65536);
  k.pe = b.take<float>((size_t)m.L * d);
  k.Wc = train ? b.take<float>((size_t)W * sW) : nullptr;
  k.G = train ? b.take<float>((size_t)W * sW) : nullptr;
  k.layer.resize(m.layers);
  for (int l = 0; l < m.layers; ++l) {
    Layer& y = k.layer[l];
    y.xin = b.take<float>((size_t)W * T * d);
    y.qkv = b.take<float>((size_t)W * T * 3 * d);
    y.P = b.take<float>((size_t)W * B * m.H * m.L * m.L);
    y.o = b.take<float>((size_t)W * T * d);
    y.xh1 = b.take<float>((size_t)W * T * d);
    y.r1 = b.take<float>((size_t)W * T);
    y.x1 = b.take<float>((size_t)W * T * d);
    y.z = b.take<float>((size_t)W * T * m.F);
    y.xh2 = b.take<float>((size_t)W * T * d);
    y.r2 = b.take<float>((size_t)W * T);
  }
  k.xf = b.take<float>((size_t)W * T * d);
  k.a = b.take<float>((size_t)W * T * d);
  k.f = b.take<float>((size_t)W * T * d);
  k.logits = b.take<float>((size_t)W * T * m.V);
  k.rloss = b.take<float>((size_t)W * T);
  k.hit = b.take<int32_t>((size_t)W * T);
  if (train) {
    k.dx = b.take<float>((size_t)W * T * d);
    k.dx1 = b.take<float>((size_t)W * T * d);
    k.dz = b.take<float>((size_t)W * T * m.F);
    k.dqkv = b.take<float>((size_t)W * T * 3 * d);
    k.dtmp = b.take<float>((size_t)W * T * d);
  } else {
    k.dx = k.dx1 = k.dz = k.dqkv = k.dtmp = nullptr;
  }
  return k;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// 1 = tcgen05 3xTF32 (default: config C 140.6 ms per iteration vs 196 ms with the SIMT
// GEMM, profiles/r02x_lm_bench_tc.log), 0 = SIMT FP32 tiled GEMM (validation)
int g_gemm_impl = 1;

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D fp32 map {inner, rows, batch} (batch stride 0 -> one batch), box {bi, br, 1}
bool map3d(CUtensorMap* map, const float* base, int64_t inner, int64_t rows, int64_t ld, int64_t batch,
           int64_t sbatch, int bi, int br, bool swz) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)(sbatch ? batch : 1)};
  const cuuint64_t strides[2] = {(cuuint64_t)ld * 4, (cuuint64_t)(sbatch ? sbatch : ld * rows) * 4};
  const cuuint32_t box[3] = {(cuuint32_t)bi, (cuuint32_t)br, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// tensor-map constraints: 16-byte aligned base and strides
bool tma_ok(const float* p, int64_t ld, int64_t sb) {
  return aligned16(p) && (ld & 3) == 0 && (sb & 3) == 0;
}

template <bool TA, bool TB, int BNT>
int launch_tc(const Gemm& g, int batch, cudaStream_t s, const char* name) {
  using Cfg = TcCfg<TA, TB, BNT>;
  CUtensorMap ma, mb;
  // A(m, k): K-major [M rows][K] (ld lda) or M-contiguous [K rows][M]; B(k, n) likewise
  const bool okA = TA ? map3d(&ma, g.A, g.M, g.K, g.lda, batch, g.sA, TCM, TCK, false)
                      : map3d(&ma, g.A, g.K, g.M, g.lda, batch, g.sA, TCK, TCM, true);
  const bool okB = TB ? map3d(&mb, g.B, g.K, g.N, g.ldb, batch, g.sB, TCK, BNT, true)
                      : map3d(&mb, g.B, g.N, g.K, g.ldb, batch, g.sB, BNT, TCK, false);
  if (!okA || !okB) {
    set_error("lm tcgen05 GEMM: cuTensorMapEncodeTiled failed");
    return FB_ERR_CUDA;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_tc_kernel<TA, TB, BNT>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    attr = true;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int64_t tiles = (int64_t)((g.N + BNT - 1) / BNT) * ((g.M + TCM - 1) / TCM) * batch;
  const int grid = (int)(tiles < sms ? tiles : sms);  // persistent: one CTA per SM
  FB_LAUNCH(name, s, (gemm_tc_kernel<TA, TB, BNT><<<grid, TC_THREADS, Cfg::SMEM, s>>>(ma, mb, g, g.sA != 0,
                                                                                        g.sB != 0, batch)));
  return launch_status(name);
}

// launch labels per caller family (0 = the LM, 1 = the ResNet): {tc nt, tc nn, tc tn, nt, nn, tn}
static const char* const kGemmNames[2][6] = {
    {"lm_gemm_tc_nt_kernel", "lm_gemm_tc_nn_kernel", "lm_gemm_tc_tn_kernel", "lm_gemm_nt_kernel", "lm_gemm_nn_kernel",
     "lm_gemm_tn_kernel"},
    {"rn_gemm_tc_nt_kernel", "rn_gemm_tc_nn_kernel", "rn_gemm_tc_tn_kernel", "rn_gemm_nt_kernel", "rn_gemm_nn_kernel",
     "rn_gemm_tn_kernel"}};

int launch_gemm(bool TA, bool TB, const Gemm& g, int batch, cudaStream_t s, int family) {
  const char* const* nm = kGemmNames[family == 1 ? 1 : 0];
  if (batch <= 0 || g.M <= 0 || g.N <= 0) return FB_OK;
  if (g_gemm_impl == 1 && g.M >= 64 && g.N >= 64 && tma_ok(g.A, g.lda, g.sA) && tma_ok(g.B, g.ldb, g.sB)) {
    // N tile 96 when it divides N (d_model-wide outputs), 64 for 64-wide outputs, else 128
    const bool n96 = g.N % 96 == 0 && g.N <= 192, n64 = g.N == 64;
    if (!TA && TB) return n96 ? launch_tc<false, true, 96>(g, batch, s, nm[0])
                          : n64 ? launch_tc<false, true, 64>(g, batch, s, nm[0])
                                : launch_tc<false, true, 128>(g, batch, s, nm[0]);
    if (!TA && !TB) return n96 ? launch_tc<false, false, 96>(g, batch, s, nm[1])
                           : n64 ? launch_tc<false, false, 64>(g, batch, s, nm[1])
                                 : launch_tc<false, false, 128>(g, batch, s, nm[1]);
    return n96 ? launch_tc<true, false, 96>(g, batch, s, nm[2])
           : n64 ? launch_tc<true, false, 64>(g, batch, s, nm[2])
                 : launch_tc<true, false, 128>(g, batch, s, nm[2]);
  }
  // 128 x 128 tiles once both output sides fill at least ~3/4 of a tile
  const bool big = g.M >= 96 && g.N >= 96;
  if (!big) {
    const dim3 grid((g.N + BN - 1) / BN, (g.M + BM - 1) / BM, batch);
    if (!TA && TB) FB_LAUNCH(nm[3], s, (gemm_kernel<false, true><<<grid, GT, 0, s>>>(g)));
    else if (!TA && !TB) FB_LAUNCH(nm[4], s, (gemm_kernel<false, false><<<grid, GT, 0, s>>>(g)));
    else FB_LAUNCH(nm[5], s, (gemm_kernel<true, false><<<grid, GT, 0, s>>>(g)));
    return launch_status("lm_gemm_kernel");
  }
  // contiguous extents: A along K (NT/NN) or M (TN); B along K (NT) or N (NN/TN)
  const int ea = TA ? g.M : g.K, eb = TB ? g.K : g.N;
  const bool vec = aligned16(g.A) && aligned16(g.B) && g.lda % 4 == 0 && g.ldb % 4 == 0 && g.sA % 4 == 0 &&
                   g.sB % 4 == 0 && ea % 4 == 0 && eb % 4 == 0;
  const dim3 grid((g.N + BN2 - 1) / BN2, (g.M + BM2 - 1) / BM2, batch);
#define FB_LM_BIG(TA_, TB_, NAME)                                                                   \
  do {                                                                                              \
    if (vec) FB_LAUNCH(NAME, s, (gemm_big_kernel<TA_, TB_, true><<<grid, GT, 0, s>>>(g)));           \
    else FB_LAUNCH(NAME, s, (gemm_big_kernel<TA_, TB_, false><<<grid, GT, 0, s>>>(g)));              \
  } while (0)
  if (!TA && TB) FB_LM_BIG(false, true, nm[3]);
  else if (!TA && !TB) FB_LM_BIG(false, false, nm[4]);
  else FB_LM_BIG(true, false, nm[5]);
#undef FB_LM_BIG
  return launch_status("lm_gemm_big_kernel");
}

Gemm gemm_base() {
  Gemm g{};
  g.alpha = 1.f;
  g.beta = 0.f;
  return g;
}

// ------------------------------------------------------------- forward
// W groups of B sentences; weights at Wc + w * sW (sW = 0: one shared theta)
int forward(const Dims& m, const Work& k, const float* Wc, int64_t sW, int W, int B, cudaStream_t s) {
  const int T = B * m.L, d = m.d;
  const LayerOff lo = layer_off(m);
  FB_LAUNCH("lm_embed_kernel", s, (embed_kernel<<<dim3(T, W), 128, 0, s>>>(k.tok, Wc, sW, k.pe, B, m.L, d,
                                                                            k.active, k.layer[0].xin)));
  int st;
  for (int l = 0; l < m.layers; ++l) {
    const Layer& y = k.layer[l];
    const float* P = Wc + layer_base(m, l);
    float* xout = l + 1 < m.layers ? k.layer[l + 1].xin : k.xf;
    Gemm g = gemm_base();  // qkv = x Wqkv^T + b
    g.A = y.xin; g.lda = d; g.sA = (int64_t)T * d;
    g.B = P + lo.in_w; g.ldb = d; g.sB = sW;
    g.C = y.qkv; g.ldc = 3 * d; g.sC = (int64_t)T * 3 * d;
    g.M = T; g.N = 3 * d; g.K = d;
    g.bias = P + lo.in_b; g.sBias = sW;
    g.active = k.active;
    if ((st = launch_gemm(false, true, g, W, s))) return st;
    FB_LAUNCH("lm_attn_fwd_kernel", s,
              (attn_fwd_kernel<<<dim3(B, W), 32 * m.H, m.L * (3 * d + 1) * sizeof(float), s>>>(
                  y.qkv, B, m.L, m.H, m.dh, k.active, y.P, y.o)));
    g = gemm_base();  // a = o Wo^T + bo
    g.A = y.o; g.lda = d; g.sA = (int64_t)T * d;
    g.B = P + lo.out_w; g.ldb = d; g.sB = sW;
    g.C = k.a; g.ldc = d; g.sC = (int64_t)T * d;
    g.M = T; g.N = d; g.K = d;
    g.bias = P + lo.out_b; g.sBias = sW;
    g.active = k.active;
    if ((st = launch_gemm(false, true, g, W, s))) return st;
    const dim3 lngrid((T + 7) / 8, W);
    FB_LAUNCH("lm_add_ln_kernel", s, (add_ln_kernel<<<lngrid, 256, 0, s>>>(y.xin, k.a, P + lo.n1_w, P + lo.n1_b, sW,
                                                                           T, d, 1e-5f, k.active, y.xh1, y.r1, y.x1)));
    g = gemm_base();  // z = x1 W1^T + b1
    g.A = y.x1; g.lda = d; g.sA = (int64_t)T * d;
    g.B = P + lo.l1_w; g.ldb = d; g.sB = sW;
    g.C = y.z; g.ldc = m.F; g.sC = (int64_t)T * m.F;
    g.M = T; g.N = m.F; g.K = d;
    g.bias = P + lo.l1_b; g.sBias = sW;
    g.active = k.active;
    if ((st = launch_gemm(false, true, g, W, s))) return st;
    g = gemm_base();  // f = relu(z) W2^T + b2
    g.A = y.z; g.lda = m.F; g.sA = (int64_t)T * m.F; g.relu_a = 1;
    g.B = P + lo.l2_w; g.ldb = m.F; g.sB = sW;
    g.C = k.f; g.ldc = d; g.sC = (int64_t)T * d;
    g.M = T; g.N = d; g.K = m.F;
    g.bias = P + lo.l2_b; g.sBias = sW;
    g.active = k.active;
    if ((st = launch_gemm(false, true, g, W, s))) return st;
    FB_LAUNCH("lm_add_ln_kernel", s, (add_ln_kernel<<<lngrid, 256, 0, s>>>(y.x1, k.f, P + lo.n2_w, P + lo.n2_b, sW,
                                                                           T, d, 1e-5f, k.active, y.xh2, y.r2, xout)));
  }
  Gemm g = gemm_base();  // logits = x E^T (tied embedding)
  g.A = k.xf; g.lda = d; g.sA = (int64_t)T * d;
  g.B = Wc; g.ldb = d; g.sB = sW;
  g.C = k.logits; g.ldc = m.V; g.sC = (int64_t)T * m.V;
  g.M = T; g.N = m.V; g.K = d;
  g.active = k.active;
  return launch_gemm(false, true, g, W, s);
}

// ------------------------------------------------------------- backward
// gradient of the step's mean loss into G (every entry written once, then the
// embedding scatter adds the input-side term)
int backward(const Dims& m, const Work& k, int64_t sW, int W, int B, cudaStream_t s, bool eval_rows = false) {
  const int T = B * m.L, d = m.d;
  const LayerOff lo = layer_off(m);
  int st;
  FB_LAUNCH("lm_ce_kernel", s, (ce_kernel<true><<<dim3(T, W), kCeT, 0, s>>>(k.logits, k.tok, B, m.L, m.V, k.nvalid,
                                                                            eval_rows ? k.rloss : nullptr,
                                                                            eval_rows ? k.hit : nullptr)));
  Gemm g = gemm_base();  // dE = dlogits^T x
  g.A = k.logits; g.lda = m.V; g.sA = (int64_t)T * m.V;
  g.B = k.xf; g.ldb = d; g.sB = (int64_t)T * d;
  g.C = k.G; g.ldc = d; g.sC = sW;
  g.M = m.V; g.N = d; g.K = T;
  g.active = k.nvalid;
  if ((st = launch_gemm(true, false, g, W, s))) return st;
  g = gemm_base();  // dx = dlogits E
  g.A = k.logits; g.lda = m.V; g.sA = (int64_t)T * m.V;
  g.B = k.Wc; g.ldb = d; g.sB = sW;
  g.C = k.dx; g.ldc = d; g.sC = (int64_t)T * d;
  g.M = T; g.N = d; g.K = m.V;
  g.active = k.nvalid;
  if ((st = launch_gemm(false, false, g, W, s))) return st;
  const dim3 lngrid((T + 7) / 8, W);
  const dim3 cs_d((d + 31) / 32, W), cs_3d((3 * d + 31) / 32, W), cs_F((m.F + 31) / 32, W);
  constexpr int CS = 32 * kCsWarps;
  for (int l = m.layers - 1; l >= 0; --l) {
    const Layer& y = k.layer[l];
    const int64_t pb = layer_base(m, l);
    const float* P = k.Wc + pb;
    float* Gl = k.G + pb;
    // LayerNorm 2: gains / biases, then into x1
    FB_LAUNCH("lm_colsum_kernel", s, (colsum_kernel<<<cs_d, CS, 0, s>>>(k.dx, y.xh2, T, d, k.nvalid, Gl + lo.n2_w, sW)));
    FB_LAUNCH("lm_colsum_kernel", s, (colsum_kernel<<<cs_d, CS, 0, s>>>(k.dx, nullptr, T, d, k.nvalid, Gl + lo.n2_b, sW)));
    FB_LAUNCH("lm_ln_bwd_kernel", s, (ln_bwd_kernel<<<lngrid, 256, 0, s>>>(k.dx, y.xh2, y.r2, P + lo.n2_w, sW, T, d,
                                                                           k.nvalid, k.dx1)));
    // feed-forward
    g = gemm_base();  // dW2 = dx1^T relu(z)
    g.A = k.dx1; g.lda = d; g.sA = (int64_t)T * d;
    g.B = y.z; g.ldb = m.F; g.sB = (int64_t)T * m.F; g.relu_b = 1;
    g.C = Gl + lo.l2_w; g.ldc = m.F; g.sC = sW;
    g.M = d; g.N = m.F; g.K = T;
    g.active = k.nvalid;
    if ((st = launch_gemm(true, false, g, W, s))) return st;
    FB_LAUNCH("lm_colsum_kernel", s, (colsum_kernel<<<cs_d, CS, 0, s>>>(k.dx1, nullptr, T, d, k.nvalid, Gl + lo.l2_b, sW)));
    g = gemm_base();  // dz = (dx1 W2) * (z > 0)
    g.A = k.dx1; g.lda = d; g.sA = (int64_t)T * d;
    g.B = P + lo.l2_w; g.ldb = m.F; g.sB = sW;
    g.C = k.dz; g.ldc = m.F; g.sC = (int64_t)T * m.F;
    g.M = T; g.N = m.F; g.K = d;
    g.aux = y.z; g.ldaux = m.F; g.sAux = (int64_t)T * m.F;
    g.active = k.nvalid;
    if ((st = launch_gemm(false, false, g, W, s))) return st;
    g = gemm_base();  // dW1 = dz^T x1
    g.A = k.dz; g.lda = m.F; g.sA = (int64_t)T * m.F;
    g.B = y.x1; g.ldb = d; g.sB = (int64_t)T * d;
    g.C = Gl + lo.l1_w; g.ldc = d; g.sC = sW;
    g.M = m.F; g.N = d; g.K = T;
    g.active = k.nvalid;
    if ((st = launch_gemm(true, false, g, W, s))) return st;
    FB_LAUNCH("lm_colsum_kernel", s, (colsum_kernel<<<cs_F, CS, 0, s>>>(k.dz, nullptr, T, m.F, k.nvalid, Gl + lo.l1_b, sW)));
    g = gemm_base();  // dx1 += dz W1
    g.A = k.dz; g.lda = m.F; g.sA = (int64_t)T * m.F;
    g.B = P + lo.l1_w; g.ldb = d; g.sB = sW;
    g.C = k.dx1; g.ldc = d; g.sC = (int64_t)T * d;
    g.M = T; g.N = d; g.K = m.F;
    g.beta = 1.f;
    g.active = k.nvalid;
    if ((st = launch_gemm(false, false, g, W, s))) return st;
    // LayerNorm 1: gains / biases, then into x and the attention output a
    FB_LAUNCH("lm_colsum_kernel", s, (colsum_kernel<<<cs_d, CS, 0, s>>>(k.dx1, y.xh1, T, d, k.nvalid, Gl + lo.n1_w, sW)));
    FB_LAUNCH("lm_colsum_kernel", s, (colsum_kernel<<<cs_d, CS, 0, s>>>(k.dx1, nullptr, T, d, k.nvalid, Gl + lo.n1_b, sW)));
    FB_LAUNCH("lm_ln_bwd_kernel", s, (ln_bwd_kernel<<<lngrid, 256, 0, s>>>(k.dx1, y.xh1, y.r1, P + lo.n1_w, sW, T, d,
                                                                           k.nvalid, k.dx)));  // dy1 -> dx
    g = gemm_base();  // dWo = dy1^T o
    g.A = k.dx; g.lda = d; g.sA = (int64_t)T * d;
    g.B = y.o; g.ldb = d; g.sB = (int64_t)T * d;
    g.C = Gl + lo.out_w; g.ldc = d; g.sC = sW;
    g.M = d; g.N = d; g.K = T;
    g.active = k.nvalid;
    if ((st = launch_gemm(true, false, g, W, s))) return st;
    FB_LAUNCH("lm_colsum_kernel", s, (colsum_kernel<<<cs_d, CS, 0, s>>>(k.dx, nullptr, T, d, k.nvalid, Gl + lo.out_b, sW)));
    g = gemm_base();  // do = dy1 Wo
    g.A = k.dx; g.lda = d; g.sA = (int64_t)T * d;
    g.B = P + lo.out_w; g.ldb = d; g.sB = sW;
    g.C = k.dtmp; g.ldc = d; g.sC = (int64_t)T * d;
    g.M = T; g.N = d; g.K = d;
    g.active = k.nvalid;
    if ((st = launch_gemm(false, false, g, W, s))) return st;
    static bool att_attr = false;
    if (!att_attr) {  // (the backward stages qkv, dO and per-head dS: > 48 KB at config C)
      cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      att_attr = true;
    }
    FB_LAUNCH("lm_attn_bwd_kernel", s,
              (attn_bwd_kernel<<<dim3(B, W), 32 * m.H,
                                 (m.L * (3 * d + 1) + m.L * (d + 1) + m.H * m.L * 33) * sizeof(float), s>>>(
                  y.qkv, y.P, k.dtmp, B, m.L, m.H, m.dh, k.nvalid, k.dqkv)));
    g = gemm_base();  // dWqkv = dqkv^T x
    g.A = k.dqkv; g.lda = 3 * d; g.sA = (int64_t)T * 3 * d;
    g.B = y.xin; g.ldb = d; g.sB = (int64_t)T * d;
    g.C = Gl + lo.in_w; g.ldc = d; g.sC = sW;
    g.M = 3 * d; g.N = d; g.K = T;
    g.active = k.nvalid;
    if ((st = launch_gemm(true, false, g, W, s))) return st;
    FB_LAUNCH("lm_colsum_kernel", s, (colsum_kernel<<<cs_3d, CS, 0, s>>>(k.dqkv, nullptr, T, 3 * d, k.nvalid,
                                                                          Gl + lo.in_b, sW)));
    g = gemm_base();  // dx (= dy1, the residual) += dqkv Wqkv
    g.A = k.dqkv; g.lda = 3 * d; g.sA = (int64_t)T * 3 * d;
    g.B = P + lo.in_w; g.ldb = d; g.sB = sW;
    g.C = k.dx; g.ldc = d; g.sC = (int64_t)T * d;
    g.M = T; g.N = d; g.K = 3 * d;
    g.beta = 1.f;
    g.active = k.nvalid;
    if ((st = launch_gemm(false, false, g, W, s))) return st;
  }
  FB_LAUNCH("lm_embed_bwd_kernel", s, (embed_bwd_kernel<<<W, 128, 0, s>>>(k.tok, k.dx, B, m.L, d, k.nvalid, k.G, sW)));
  return launch_status("lm backward");
}

bool dims_ok(const Dims& m) {
  const size_t att = (size_t)(m.L * (3 * m.d + 1) + m.L * (m.d + 1) + m.H * m.L * 33) * sizeof(float);
  return m.V >= 2 && m.d >= 1 && m.d <= 256 && m.H >= 1 && m.H <= 16 && m.d % m.H == 0 && m.dh <= 32 &&
         m.F >= 1 && m.layers >= 1 && m.L >= 1 && m.L <= 32 && att <= 200 * 1024;
}

Dims parse(const int32_t* dims) {
  Dims m;
  m.V = dims[0];
  m.d = dims[1];
  m.H = dims[2] > 0 ? dims[2] : 1;
  m.dh = m.d / m.H;
  m.F = dims[3];
  m.layers = dims[4];
  m.L = dims[5];
  return m;
}

}  // namespace lm
}  // namespace fb

extern "C" {

int fb_lm_set_gemm_impl(int impl) {
  FB_REQUIRE(impl == 0 || impl == 1, "lm_set_gemm_impl: 0 (SIMT FP32) or 1 (tcgen05 3xTF32, default)");
  fb::lm::g_gemm_impl = impl;
  return FB_OK;
}

int64_t fb_lm_num_params(const int32_t* dims) { return dims ? fb::lm::num_params(fb::lm::parse(dims)) : 0; }

int64_t fb_lm_workspace_bytes(const int32_t* dims, int batch_size, int clients_per_wave, int eval_groups) {
  if (!dims || batch_size < 1) return 0;
  const fb::lm::Dims m = fb::lm::parse(dims);
  fb::lm::Buf a, b;
  fb::lm::carve(m, clients_per_wave > 0 ? clients_per_wave : 1, batch_size, true, a);
  fb::lm::carve(m, eval_groups > 0 ? eval_groups : 1, batch_size, false, b);
  return (int64_t)(a.off > b.off ? a.off : b.off) + 256;
}

int fb_eval_lm_f32(const float* theta, const int32_t* dims, const float* X, const int64_t* row_start,
                   const int32_t* num_rows, const int32_t* h_num_rows, int num_clients, double* loss_sum,
                   int32_t* correct, int batch_size, int eval_groups, void* workspace, int64_t workspace_bytes,
                   const int32_t* perms, const int64_t* perm_off, int skip, void* stream) {
  FB_REQUIRE(dims != nullptr && h_num_rows != nullptr, "eval_lm: null dims / host row counts");
  const fb::lm::Dims m = fb::lm::parse(dims);
  FB_UNSUPPORTED(fb::lm::dims_ok(m), "eval_lm: unsupported shape (d <= 256, d %% heads == 0, head dim <= 32, seq <= 32)");
  FB_REQUIRE(num_clients >= 0 && num_clients <= 65536 && batch_size >= 1 && eval_groups >= 1,
             "eval_lm: bad sizes");
  FB_REQUIRE(workspace_bytes >= fb_lm_workspace_bytes(dims, batch_size, 1, eval_groups), "eval_lm: workspace too small");
  cudaStream_t s = fb::as_stream(stream);
  if (num_clients == 0) return FB_OK;
  cudaMemsetAsync(loss_sum, 0, sizeof(double) * num_clients, s);
  cudaMemsetAsync(correct, 0, sizeof(int32_t) * num_clients, s);
  fb::lm::Buf b;
  b.base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
  const fb::lm::Work k = fb::lm::carve(m, eval_groups, batch_size, false, b);
  const int W = eval_groups, B = batch_size, L = m.L;
  FB_LAUNCH("lm_positions_kernel", s, (fb::lm::positions_kernel<<<(L * m.d + 255) / 256, 256, 0, s>>>(k.pe, L, m.d)));
  FB_LAUNCH("lm_ones_kernel", s, (fb::lm::ones_kernel<<<(W + 255) / 256, 256, 0, s>>>(k.active, W)));
  FB_REQUIRE(!perms || (perm_off && skip >= 0), "eval_lm: perms need perm_off and skip >= 0");
  const int sk = perms ? skip : 0;
  FB_LAUNCH("lm_sent_offsets_kernel", s, (fb::lm::sent_offsets_kernel<<<1, 32, 0, s>>>(num_rows, num_clients, k.sent_off, sk)));
  int64_t total = 0;
  for (int c = 0; c < num_clients; ++c) total += h_num_rows[c] - (sk < h_num_rows[c] ? sk : h_num_rows[c]);
  const int chunk = W * B;
  for (int64_t g0 = 0; g0 < total; g0 += chunk) {
    const int cnt = (int)(total - g0 < chunk ? total - g0 : chunk);
    FB_LAUNCH("lm_gather_eval_kernel", s, (fb::lm::gather_eval_kernel<<<chunk, 32, 0, s>>>(
                                              X, row_start, k.sent_off, num_clients, g0, cnt, L, k.tok, perms,
                                              perm_off, num_rows, sk)));
    int st = fb::lm::forward(m, k, theta, 0, W, B, s);
    if (st) return st;
    FB_LAUNCH("lm_ce_kernel", s, (fb::lm::ce_kernel<false><<<dim3(B * L, W), fb::lm::kCeT, 0, s>>>(
                                     k.logits, k.tok, B, L, m.V, nullptr, k.rloss, k.hit)));
    FB_LAUNCH("lm_eval_accum_kernel", s, (fb::lm::eval_accum_kernel<<<(num_clients + 127) / 128, 128, 0, s>>>(
                                             k.rloss, k.hit, k.sent_off, num_rows, num_clients, g0, cnt, L, loss_sum,
                                             correct, sk)));
  }
  return fb::launch_status("eval_lm");
}

int fb_local_sgd_lm_f32(const float* theta_t, const int32_t* dims, const float* X, const int64_t* row_start,
                        const int32_t* num_rows, const int32_t* h_num_rows, const int32_t* perms,
                        const int64_t* perm_off, int num_clients, int epochs, int batch_size, float lr,
                        float prox_mu, const float* control, int64_t ld_control, float* delta_out, int64_t ld_delta,
                        int32_t* nonfinite, int clients_per_wave, void* workspace, int64_t workspace_bytes,
                        double* eval_loss, int32_t* eval_correct, void* stream) {
  FB_REQUIRE(dims != nullptr && h_num_rows != nullptr, "local_sgd_lm: null dims / host row counts");
  const fb::lm::Dims m = fb::lm::parse(dims);
  FB_UNSUPPORTED(fb::lm::dims_ok(m), "local_sgd_lm: unsupported shape (d <= 256, d %% heads == 0, head dim <= 32, seq <= 32)");
  const int64_t D = fb::lm::num_params(m);
  FB_REQUIRE(num_clients >= 0 && epochs >= 0 && batch_size >= 1 && clients_per_wave >= 1 && ld_delta >= D,
             "local_sgd_lm: bad sizes");
  FB_REQUIRE(workspace_bytes >= fb_lm_workspace_bytes(dims, batch_size, clients_per_wave, 1),
             "local_sgd_lm: workspace too small");
  cudaStream_t s = fb::as_stream(stream);
  if (num_clients == 0) return FB_OK;
  fb::lm::Buf b;
  b.base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
  fb::lm::Work k = fb::lm::carve(m, clients_per_wave, batch_size, true, b);
  const int64_t sW = (D + 3) & ~int64_t(3);
  const int B = batch_size, L = m.L;
  FB_LAUNCH("lm_positions_kernel", s, (fb::lm::positions_kernel<<<(L * m.d + 255) / 256, 256, 0, s>>>(k.pe, L, m.d)));
  for (int c0 = 0; c0 < num_clients; c0 += clients_per_wave) {
    const int W = num_clients - c0 < clients_per_wave ? num_clients - c0 : clients_per_wave;
    int max_steps = 0;
    for (int c = c0; c < c0 + W; ++c) {
      const int n = h_num_rows[c];
      const int st = n > 0 ? epochs * ((n + B - 1) / B) : 0;
      max_steps = st > max_steps ? st : max_steps;
    }
    float* Dl = delta_out + (int64_t)c0 * ld_delta;
    FB_LAUNCH("lm_init_wave_kernel", s, (fb::lm::init_wave_kernel<<<dim3(256, W), 256, 0, s>>>(theta_t, D, k.Wc, sW,
                                                                                                Dl, ld_delta)));
    for (int step = 0; step < max_steps; ++step) {
      FB_LAUNCH("lm_gather_batch_kernel", s, (fb::lm::gather_batch_kernel<<<W, 128, 0, s>>>(
                                                 X, row_start, num_rows, perms, perm_off, c0, epochs, B, L, step,
                                                 k.tok, k.nvalid)));
      k.active = k.nvalid;  // (nonzero = the client has a minibatch this step)
      int st = fb::lm::forward(m, k, k.Wc, sW, W, B, s);
      if (st) return st;
      const bool ev0 = step == 0 && eval_loss != nullptr;  // step 0 runs at theta_t: the batch's evaluation
      st = fb::lm::backward(m, k, sW, W, B, s, ev0);
      if (st) return st;
      if (ev0)
        FB_LAUNCH("lm_step0_eval_kernel", s, (fb::lm::step0_eval_kernel<<<(W + 127) / 128, 128, 0, s>>>(
                                                 k.rloss, k.hit, k.nvalid, W, B, L, eval_loss + c0, eval_correct + c0)));
      FB_LAUNCH("lm_sgd_kernel", s, (fb::lm::sgd_kernel<<<dim3(128, W), 256, 0, s>>>(
                                        k.Wc, k.G, sW, Dl, ld_delta,
                                        control ? control + (ld_control ? (int64_t)c0 * ld_control : 0) : nullptr,
                                        ld_control, D, lr, prox_mu, k.nvalid)));
    }
    FB_LAUNCH("lm_nonfinite_kernel", s, (fb::lm::nonfinite_kernel<<<W, 256, 0, s>>>(Dl, ld_delta, D, nonfinite + c0)));
  }
  return fb::launch_status("local_sgd_lm");
}

}  // extern "C"
