// Config D: the FLAIR-shaped ResNet-18 with GroupNorm and a multi-label sigmoid
// BCE (models.ResNet18), local SGD of a
// whole cohort at once and the pre-training evaluation.
//
// The reference has no ResNet: the arithmetic is the oracle's ResNet18
// (oracle/port.py, pinned to float64 autograd), trained through the reference's
// generic update rule (fedsim/models/models.py:53-79):
//   theta <- theta - lr * (grad + prox_mu * (theta - theta_t) + control),
// batches in perms order, the tail batch kept, the batch loss the mean over the
// batch's images of each image's mean BCE over its K labels.
//
// Layout.  A wave of W clients is trained together, every client's step-s
// minibatch of B images side by side; activations are NHWC fp32 [W][B][H][W][C]
// (a conv's GEMM output [B*H*W, C_out] IS the next activation), each client's
// weights a row of Wc [W, D] and its gradient a row of G [W, D] in
// ResNet18.param_dims order (PyTorch OIHW conv weights).  Clients are assigned
// to waves largest-first (the within-GPU form of the reference's LPT scheduler,
// fedsim/engine/scheduling.py:54-78), so a wave's clients run similar numbers
// of local steps.  Per conv: an im2col gather in (ky, kx, c) column order --
// channel-contiguous on both sides, so reads of the NHWC source and writes of the
// col rows are float4-coalesced -- and one grouped GEMM over the wave on the
// tcgen05 3xTF32 kernel (grouped_gemm.cuh): forward Y = col Wp^T, backward
// dWp = dY^T col and dcol = dY Wp followed by a deterministic col2im gather.  Wp
// is the step's conv weights permuted once from OIHW to O(HW)I (all convs in one
// launch); the dWp blocks are permuted back into G's OIHW rows in one launch.  GroupNorm: per-chunk
// fp64 partial sums, a warp-per-(image, group) finalize in fixed order, and an
// elementwise apply fused with the residual add and the ReLU; its backward is
// the same three-phase shape.  Every reduction has a fixed order, so reruns are
// bit-identical.  Images are read straight from the population rows (CHW
// pixels, then the K label indicators) through a per-slot row index.

#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <numeric>
#include <vector>

#include "fb_common.cuh"
#include "grouped_gemm.cuh"

namespace fb {
namespace rn {

using lm::Gemm;
using lm::gemm_base;
inline int rn_gemm(bool TA, bool TB, const Gemm& g, int batch, cudaStream_t s) {
  return lm::launch_gemm(TA, TB, g, batch, s, 1);  // (launch labels rn_gemm_*)
}

constexpr float kEps = 1e-5f;
constexpr int kT = 256;                // threads of the elementwise / partial-sum kernels
constexpr int kChunkElems = 16384;     // elements per GroupNorm partial-sum CTA

struct Dims {
  int K, w, G, S;  // classes, width, norm groups, image side
};

struct Conv {
  int ci, co, k, stride, pad, hin, hout;
  int64_t w_off;  // OIHW weights in the parameter row
  int64_t p_off;  // O(HW)I weights (rows of kp) in the permuted buffer
  int kk() const { return ci * k * k; }
  int kp() const { return (kk() + 3) & ~3; }  // im2col row stride (16-byte rows for TMA)
  int pin() const { return hin * hin; }
  int pout() const { return hout * hout; }
};
struct Norm {
  int c;
  int64_t g_off, b_off;
};
struct Block {
  Conv c1, c2, ds;
  Norm n1, n2, nd;
  bool has_ds;
};
struct Net {
  Dims m;
  Conv stem;
  Norm n0;
  int hs, hp;  // stem conv output side, maxpool output side
  Block blk[8];
  int64_t fc_w, fc_b, D;
  int64_t P;  // permuted-weight floats per client
  int nconv;
  Conv convs[24];  // every conv, for the permutation launches
};

inline int out_side(int h, int k, int s, int p) { return (h + 2 * p - k) / s + 1; }

inline Net build(const Dims& m) {
  Net n;
  n.m = m;
  int64_t o = 0, po = 0;
  n.nconv = 0;
  auto conv = [&](int ci, int co, int k, int s, int p, int hin) {
    Conv c{ci, co, k, s, p, hin, out_side(hin, k, s, p), o, po};
    o += (int64_t)co * ci * k * k;
    po += (int64_t)co * c.kp();
    n.convs[n.nconv++] = c;
    return c;
  };
  auto norm = [&](int c) {
    Norm q{c, o, o + c};
    o += 2 * c;
    return q;
  };
  n.stem = conv(3, m.w, 7, 2, 3, m.S);
  n.n0 = norm(m.w);
  n.hs = n.stem.hout;
  n.hp = out_side(n.hs, 3, 2, 1);
  int cin = m.w, h = n.hp;
  for (int st = 0; st < 4; ++st) {
    const int cout = m.w << st;
    for (int b = 0; b < 2; ++b) {
      const int s = (st > 0 && b == 0) ? 2 : 1;
      Block& k = n.blk[st * 2 + b];
      k.c1 = conv(cin, cout, 3, s, 1, h);
      k.n1 = norm(cout);
      k.c2 = conv(cout, cout, 3, 1, 1, k.c1.hout);
      k.n2 = norm(cout);
      k.has_ds = s != 1 || cin != cout;
      if (k.has_ds) {
        k.ds = conv(cin, cout, 1, s, 0, h);
        k.nd = norm(cout);
      } else {
        k.ds = Conv{};
        k.nd = Norm{};
      }
      cin = cout;
      h = k.c1.hout;
    }
  }
  n.fc_w = o;
  o += (int64_t)m.K * 8 * m.w;
  n.fc_b = o;
  o += m.K;
  n.D = o;
  n.P = po;
  return n;
}

inline bool pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

inline bool dims_ok(const Dims& m) {
  // channels: powers of two <= 512 (the partial-sum kernels' channel mapping); groups divide them
  return m.K >= 1 && m.K <= 256 && pow2(m.w) && m.w >= 4 && m.w <= 64 && m.G >= 1 && m.w % m.G == 0 &&
         m.S >= 32 && m.S <= 1024;
}

inline Dims parse(const int32_t* d) { return Dims{d[0], d[1], d[2], d[3]}; }

// weight-gradient K split: the GEMM's K is B * P_out rows; long ones (the stem, layer 1)
// are cut into S power-of-two chunks of >= 2048 rows so (client, chunk) tiles fill the SMs
inline int ksplit(int rows) {
  int S = 1;
  while (S < 16 && rows % (2 * S) == 0 && rows / (2 * S) >= 2048) S *= 2;
  return S;
}

inline int nchunks(int P, int C) {
  const int per = std::max(1, kChunkElems / C);  // pixels per chunk
  return (P + per - 1) / per;
}

// ------------------------------------------------------------ batch gather
// Slot (w, i) of the wave: client c = ord[c0 + w]; step s -> epoch e = s / nb, batch
// j = s % nb; image perms[c][e * n + j * B + i] (row -1 past the batch).  Labels copied
// into lab[w][i][K]; nvalid[w] = images in the batch (0: client idle this step).
__global__ void gather_batch_kernel(const float* __restrict__ X, int64_t ldx, int64_t lab_off, int K,
                                    const int64_t* __restrict__ row_start, const int32_t* __restrict__ num_rows,
                                    const int32_t* __restrict__ perms, const int64_t* __restrict__ perm_off,
                                    const int32_t* __restrict__ ord, int c0, int epochs, int B, int step,
                                    int64_t* __restrict__ rows, float* __restrict__ lab,
                                    int32_t* __restrict__ nvalid) {
  const int w = blockIdx.x, c = ord[c0 + w];
  const int n = num_rows[c];
  const int nb = n > 0 ? (n + B - 1) / B : 0;
  const bool live = nb > 0 && step < epochs * nb;
  const int e = live ? step / nb : 0, j = live ? step % nb : 0;
  const int cnt = live ? min(B, n - j * B) : 0;
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    int64_t r = -1;
    if (i < cnt) r = row_start[c] + perms[perm_off[c] + (int64_t)e * n + j * B + i];
    rows[(int64_t)w * B + i] = r;
  }
  for (int q = threadIdx.x; q < B * K; q += blockDim.x) {
    const int i = q / K, k = q - i * K;
    float v = 0.f;
    if (i < cnt) {
      const int64_t r = row_start[c] + perms[perm_off[c] + (int64_t)e * n + j * B + i];
      v = X[r * ldx + lab_off + k];
    }
    lab[(int64_t)w * B * K + q] = v;
  }
  if (threadIdx.x == 0) nvalid[w] = cnt;
}

// eval chunk: images [g0, g0 + cnt) of the cohort in client-major order, slot i -> (w, b)
// (perms != nullptr: client c's evaluated images are epoch 0's perms[perm_off[c] + skip_c ..])
__global__ void gather_eval_kernel(const float* __restrict__ X, int64_t ldx, int64_t lab_off, int K,
                                   const int64_t* __restrict__ row_start, const int64_t* __restrict__ img_off, int C,
                                   int64_t g0, int cnt, int total_slots, const int32_t* __restrict__ perms,
                                   const int64_t* __restrict__ perm_off, const int32_t* __restrict__ num_rows,
                                   int skip, int64_t* __restrict__ rows, float* __restrict__ lab) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total_slots) return;
  int64_t r = -1;
  if (i < cnt) {
    const int64_t g = g0 + i;
    int lo = 0, hi = C - 1;  // last client with img_off <= g
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (img_off[mid] <= g) lo = mid;
      else hi = mid - 1;
    }
    const int64_t j = g - img_off[lo];
    r = row_start[lo] + (perms ? perms[perm_off[lo] + min(skip, num_rows[lo]) + j] : j);
  }
  rows[i] = r;
  for (int k = 0; k < K; ++k) lab[(int64_t)i * K + k] = r >= 0 ? X[r * ldx + lab_off + k] : 0.f;
}

__global__ void img_offsets_kernel(const int32_t* __restrict__ num_rows, int C, int64_t* __restrict__ off, int skip) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int64_t s = 0;
    for (int c = 0; c < C; ++c) {
      off[c] = s;
      s += num_rows[c] - min(skip, num_rows[c]);
    }
  }
}

// ------------------------------------------------------------------ im2col
// col[w][(b, oy, ox)][q], q = (ky k + kx) ci + c < ci k^2, zero in the padding columns
// up to kp; source NHWC [w][b][hin][hin][ci].  A CTA fills kRows consecutive col rows;
// the per-column (ky, kx, c) and per-row (b, iy0, ix0) decodings are tabulated in
// shared memory once, and consecutive threads take consecutive columns (4 channels
// each when ci % 4 == 0), so source reads and col writes are contiguous channel runs.
constexpr int kRows = 32;
constexpr int kMaxQ = 1280;  // columns / V per row (kp <= 5120)

template <bool kVec>
__global__ void __launch_bounds__(256) im2col_kernel(const float* __restrict__ src, int64_t s_src, int B, int ci,
                                                     int hin, int k, int stride, int pad, int hout, int kp,
                                                     const int32_t* __restrict__ active, float* __restrict__ col,
                                                     int64_t s_col) {
  const int w = blockIdx.y;
  if (active && !active[w]) return;
  constexpr int V = kVec ? 4 : 1;
  __shared__ int2 tab[kMaxQ];
  __shared__ int4 rinfo[kRows];
  const int kc = ci * k * k, po = hout * hout, Q = kp / V;
  for (int q4 = threadIdx.x; q4 < Q; q4 += blockDim.x) {
    const int q = q4 * V;
    if (q < kc) {
      const int t = q / ci, c = q - t * ci, ky = t / k;
      tab[q4] = make_int2((ky << 16) | (t - ky * k), c);
    } else {
      tab[q4] = make_int2(-1, 0);
    }
  }
  const int64_t rows = (int64_t)B * po;
  float* out = col + (int64_t)w * s_col;
  const float* sb = src + (int64_t)w * s_src;
  for (int64_t r0 = (int64_t)blockIdx.x * kRows; r0 < rows; r0 += (int64_t)gridDim.x * kRows) {
    __syncthreads();
    if (threadIdx.x < kRows) {
      const int64_t r = r0 + threadIdx.x;
      const int b = (int)(r / po), pix = (int)(r - (int64_t)b * po);
      const int oy = pix / hout, ox = pix - oy * hout;
      rinfo[threadIdx.x] = make_int4(b, oy * stride - pad, ox * stride - pad, r < rows);
    }
    __syncthreads();
    const int nr = (int)(rows - r0 < kRows ? rows - r0 : kRows);
    for (int j = threadIdx.x; j < nr * Q; j += blockDim.x) {
      const int rr = j / Q, q4 = j - rr * Q;
      const int2 tq = tab[q4];
      const int4 ri = rinfo[rr];
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (tq.x >= 0) {
        const int iy = ri.y + (tq.x >> 16), ix = ri.z + (tq.x & 0xffff);
        if (iy >= 0 && iy < hin && ix >= 0 && ix < hin) {
          const float* p = sb + (((int64_t)ri.x * hin + iy) * hin + ix) * ci + tq.y;
          if (kVec) v = *reinterpret_cast<const float4*>(p);
          else v.x = *p;
        }
      }
      float* o = out + (r0 + rr) * kp + q4 * V;
      if (kVec) *reinterpret_cast<float4*>(o) = v;
      else *o = v.x;
    }
  }
}

// the stem's input: batch images from the population rows (CHW) into NHWC [w][b][S][S][3]
__global__ void stem_input_kernel(const float* __restrict__ X, int64_t ldx, const int64_t* __restrict__ rows, int B,
                                  int S, const int32_t* __restrict__ active, float* __restrict__ out) {
  const int w = blockIdx.y;
  if (active && !active[w]) return;
  const int64_t per = (int64_t)S * S, total = (int64_t)B * per * 3;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % 3);
    const int64_t pix = i / 3;
    const int b = (int)(pix / per);
    const int64_t yx = pix - (int64_t)b * per;
    const int64_t row = rows[(int64_t)w * B + b];
    out[(int64_t)w * total + i] = row >= 0 ? X[row * ldx + c * per + yx] : 0.f;
  }
}

// dx[w][b][y][x][c] (=|+=) sum of the dcol entries that read it (+ add * (mask > 0));
// one thread per (input pixel, 4 channels), the tap loops unrolled for the conv's
// (K, S) (3x3/1, 3x3/2, 1x1/2), dcol rows read as contiguous channel runs
template <int K, int S>
__global__ void __launch_bounds__(256) col2im_kernel(const float* __restrict__ dcol, int64_t s_col, int ldcol, int B,
                                                     int ci, int hin, int pad, int hout,
                                                     const int32_t* __restrict__ active,
                                                     const float* __restrict__ add, const float* __restrict__ mask,
                                                     int accumulate, float* __restrict__ dx, int64_t s_dx) {
  const int w = blockIdx.y;
  if (active && !active[w]) return;
  const int pin = hin * hin, c4n = ci >> 2;
  const int64_t total = (int64_t)B * pin * c4n;
  const float* dc = dcol + (int64_t)w * s_col;
  float* o = dx + (int64_t)w * s_dx;
  const float* ad = add ? add + (int64_t)w * s_dx : nullptr;
  const float* mk = mask ? mask + (int64_t)w * s_dx : nullptr;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % c4n) * 4;
    const int64_t pix = i / c4n;
    const int b = (int)(pix / pin);
    const int rem = (int)(pix - (int64_t)b * pin);
    const int y = rem / hin, x = rem - y * hin;
    const float* db = dc + (int64_t)b * hout * hout * ldcol + c;
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int ky = 0; ky < K; ++ky) {
      const int ty = y + pad - ky;
      if (ty < 0 || (S > 1 && (ty % S))) continue;
      const int oy = ty / S;
      if (oy >= hout) continue;
#pragma unroll
      for (int kx = 0; kx < K; ++kx) {
        const int tx = x + pad - kx;
        if (tx < 0 || (S > 1 && (tx % S))) continue;
        const int ox = tx / S;
        if (ox >= hout) continue;
        const float4 v = *reinterpret_cast<const float4*>(db + (int64_t)(oy * hout + ox) * ldcol + (ky * K + kx) * ci);
        s.x += v.x;
        s.y += v.y;
        s.z += v.z;
        s.w += v.w;
      }
    }
    const int64_t e = pix * ci + c;
    if (ad) {
      const float4 a = *reinterpret_cast<const float4*>(ad + e);
      if (mk) {
        const float4 m = *reinterpret_cast<const float4*>(mk + e);
        s.x += m.x > 0.f ? a.x : 0.f;
        s.y += m.y > 0.f ? a.y : 0.f;
        s.z += m.z > 0.f ? a.z : 0.f;
        s.w += m.w > 0.f ? a.w : 0.f;
      } else {
        s.x += a.x;
        s.y += a.y;
        s.z += a.z;
        s.w += a.w;
      }
    }
    if (accumulate) {
      const float4 p = *reinterpret_cast<const float4*>(o + e);
      s.x += p.x;
      s.y += p.y;
      s.z += p.z;
      s.w += p.w;
    }
    *reinterpret_cast<float4*>(o + e) = s;
  }
}

// every conv's weights OIHW (parameter row) <-> O(HW)I rows of kp (permuted buffer);
// to_perm: Wp <- W (padding columns 0), else G <- dWp.  One thread per permuted entry.
struct ConvTable {
  int n;
  int64_t w_off[24], p_off[24];
  int co[24], ci[24], kk[24], kp[24];
};

__global__ void permute_kernel(ConvTable tb, int64_t P, const float* __restrict__ W, int64_t sW,
                               float* __restrict__ Wp, int64_t sP, const int32_t* __restrict__ active, int to_perm) {
  const int w = blockIdx.y, j = blockIdx.z;  // client slot, conv
  if (active && !active[w]) return;
  const int kp = tb.kp[j], ci = tb.ci[j], kk = tb.kk[j];
  const int n = tb.co[j] * kp;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int64_t i = tb.p_off[j] + e;
    const int o = e / kp, q = e - o * kp;
    if (q >= ci * kk) {
      if (to_perm) Wp[(int64_t)w * sP + i] = 0.f;
      continue;
    }
    const int t = q / ci, c = q - t * ci;
    const int64_t src = tb.w_off[j] + ((int64_t)o * ci + c) * kk + t;
    if (to_perm) Wp[(int64_t)w * sP + i] = W[(int64_t)w * sW + src];
    else  // (W = the transposed gradient blocks dWp^T [kp][co], Wp = G here)
      Wp[(int64_t)w * sW + src] = W[(int64_t)w * sP + tb.p_off[j] + (int64_t)q * tb.co[j] + o];
  }
}

// --------------------------------------------------------------- GroupNorm
// Partial sums over chunks of an image's pixels (all channels), fp64.  Element i of
// the chunk's contiguous [p0 * C, p1 * C) range has channel i % C; thread t owns the
// channels t % C (C <= 256) or t + 256 j (C = 512).
template <int NA>
__device__ __forceinline__ int chan_of(int t, int j, int C) {
  return NA == 1 ? (t % C) : t + 256 * j;
}

// forward: part[w][b][chunk][g] = {sum x, sum x^2}
template <int NA>
__global__ void __launch_bounds__(kT) gn_stats_kernel(const float* __restrict__ x, int64_t s_x, int P, int C, int G,
                                                      int chunk, int nch, const int32_t* __restrict__ active,
                                                      double2* __restrict__ part) {
  const int w = blockIdx.z, b = blockIdx.y, ch = blockIdx.x, t = threadIdx.x;
  if (active && !active[w]) return;
  const int B = gridDim.y;
  const int p0 = ch * chunk, p1 = min(P, p0 + chunk);
  const float* xb = x + (int64_t)w * s_x + (int64_t)b * P * C;
  double s[NA], q[NA];
#pragma unroll
  for (int j = 0; j < NA; ++j) s[j] = q[j] = 0.0;
  const int64_t e0 = (int64_t)p0 * C, e1 = (int64_t)p1 * C;
  for (int64_t i = e0 + t; i < e1; i += kT) {
    const double v = xb[i];
    const int j = NA == 1 ? 0 : (int)((i / 256) % NA);
    s[j] += v;
    q[j] += v * v;
  }
  __shared__ double2 sh[kT * NA];
#pragma unroll
  for (int j = 0; j < NA; ++j) sh[t * NA + j] = make_double2(s[j], q[j]);
  __syncthreads();
  // per group, fixed order: channels of the group, then the lanes holding each channel
  const int Cg = C / G;
  for (int g = t; g < G; g += kT) {
    double a = 0.0, bq = 0.0;
    for (int c = g * Cg; c < (g + 1) * Cg; ++c) {
      if (NA == 1) {
        for (int l = c; l < kT; l += C) {
          a += sh[l].x;
          bq += sh[l].y;
        }
      } else {
        const int l = c % 256, j = c / 256;
        a += sh[l * NA + j].x;
        bq += sh[l * NA + j].y;
      }
    }
    part[(((int64_t)w * B + b) * nch + ch) * G + g] = make_double2(a, bq);
  }
}

// mean / rstd per (w, b, g): a warp per (b, g), lanes over chunks, fixed shuffle tree
__global__ void gn_finalize_kernel(const double2* __restrict__ part, int B, int G, int nch, double n,
                                   const int32_t* __restrict__ active, float2* __restrict__ stats) {
  const int w = blockIdx.y;
  if (active && !active[w]) return;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (gw >= B * G) return;
  const int b = gw / G, g = gw - b * G;
  double a = 0.0, q = 0.0;
  for (int ch = lane; ch < nch; ch += 32) {
    const double2 v = part[(((int64_t)w * B + b) * nch + ch) * G + g];
    a += v.x;
    q += v.y;
  }
  a = warp_sum(a);
  q = warp_sum(q);
  if (lane == 0) {
    const double mean = a / n;
    const double var = fmax(q / n - mean * mean, 0.0);
    stats[((int64_t)w * B + b) * G + g] = make_float2((float)mean, (float)(1.0 / sqrt(var + (double)kEps)));
  }
}

// y = (x - mean) rstd gamma + beta (+ res) (ReLU); 4 channels per thread (C is a power of
// two >= 4), 32-bit indices within the image
__global__ void __launch_bounds__(kT) gn_apply_kernel(const float* __restrict__ x, int64_t s_x, int P, int C, int G,
                                                      const float2* __restrict__ stats, const float* __restrict__ Wc,
                                                      int64_t sW, int64_t g_off, int64_t b_off,
                                                      const float* __restrict__ res, int relu,
                                                      const int32_t* __restrict__ active, float* __restrict__ y) {
  const int w = blockIdx.y;
  if (active && !active[w]) return;
  const int B = gridDim.z;
  const int b = blockIdx.z;
  const int Cg = C / G;
  const float* gam = Wc + (int64_t)w * sW + g_off;
  const float* bet = Wc + (int64_t)w * sW + b_off;
  const int64_t base = (int64_t)w * s_x + (int64_t)b * P * C;
  const float2* st = stats + ((int64_t)w * B + b) * G;
  const float4* xv = reinterpret_cast<const float4*>(x + base);
  const float4* rv = res ? reinterpret_cast<const float4*>(res + base) : nullptr;
  float4* yv = reinterpret_cast<float4*>(y + base);
  const int n4 = P * C / 4;
  for (int i = blockIdx.x * kT + threadIdx.x; i < n4; i += gridDim.x * kT) {
    const int c = (4 * i) & (C - 1);
    const float4 v = xv[i];
    float o[4] = {v.x, v.y, v.z, v.w};
    float4 r = rv ? rv[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 ms = st[(c + e) / Cg];
      float q = (o[e] - ms.x) * ms.y * gam[c + e] + bet[c + e];
      if (rv) q += rr[e];
      o[e] = relu ? fmaxf(q, 0.f) : q;
    }
    yv[i] = make_float4(o[0], o[1], o[2], o[3]);
  }
}

// backward partials: dv = dout * (mask > 0) (mask nullable), xhat = (x - mean) rstd;
// part[w][b][chunk][c] = {sum dv, sum dv xhat}
template <int NA>
__global__ void __launch_bounds__(kT) gn_bwd_stats_kernel(const float* __restrict__ dout,
                                                          const float* __restrict__ mask,
                                                          const float* __restrict__ x, int64_t s_x, int P, int C,
                                                          int G, const float2* __restrict__ stats, int chunk, int nch,
                                                          const int32_t* __restrict__ active,
                                                          double2* __restrict__ part) {
  const int w = blockIdx.z, b = blockIdx.y, ch = blockIdx.x, t = threadIdx.x;
  if (active && !active[w]) return;
  const int B = gridDim.y;
  const int Cg = C / G;
  const int p0 = ch * chunk, p1 = min(P, p0 + chunk);
  const int64_t base = (int64_t)w * s_x + (int64_t)b * P * C;
  const float2* st = stats + ((int64_t)w * B + b) * G;
  double s[NA], q[NA];
#pragma unroll
  for (int j = 0; j < NA; ++j) s[j] = q[j] = 0.0;
  const int64_t e0 = (int64_t)p0 * C, e1 = (int64_t)p1 * C;
  for (int64_t i = e0 + t; i < e1; i += kT) {
    const int j = NA == 1 ? 0 : (int)((i / 256) % NA);
    const int c = chan_of<NA>(t, j, C);
    float dv = dout[base + i];
    if (mask && !(mask[base + i] > 0.f)) dv = 0.f;
    const float2 ms = st[c / Cg];
    const float xh = (x[base + i] - ms.x) * ms.y;
    s[j] += (double)dv;
    q[j] += (double)dv * (double)xh;
  }
  __shared__ double2 sh[kT * NA];
#pragma unroll
  for (int j = 0; j < NA; ++j) sh[t * NA + j] = make_double2(s[j], q[j]);
  __syncthreads();
  for (int c = t; c < C; c += kT) {
    double a = 0.0, bq = 0.0;
    if (NA == 1) {
      for (int l = c; l < kT; l += C) {
        a += sh[l].x;
        bq += sh[l].y;
      }
    } else {
      a = sh[(c % 256) * NA + c / 256].x;
      bq = sh[(c % 256) * NA + c / 256].y;
    }
    part[(((int64_t)w * B + b) * nch + ch) * C + c] = make_double2(a, bq);
  }
}

// per (w, b, g): coef = {sum_g gamma dv / n, sum_g gamma dv xhat / n}; warp per (b, g)
__global__ void gn_bwd_finalize_kernel(const double2* __restrict__ part, int B, int C, int G, int nch, double n,
                                       const float* __restrict__ Wc, int64_t sW, int64_t g_off,
                                       const int32_t* __restrict__ active, float2* __restrict__ coef) {
  const int w = blockIdx.y;
  if (active && !active[w]) return;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (gw >= B * G) return;
  const int b = gw / G, g = gw - b * G, Cg = C / G;
  const float* gam = Wc + (int64_t)w * sW + g_off;
  double a = 0.0, q = 0.0;
  for (int e = lane; e < Cg * nch; e += 32) {
    const int ch = e / Cg, c = g * Cg + (e - ch * Cg);
    const double2 v = part[(((int64_t)w * B + b) * nch + ch) * C + c];
    a += (double)gam[c] * v.x;
    q += (double)gam[c] * v.y;
  }
  a = warp_sum(a);
  q = warp_sum(q);
  if (lane == 0) coef[((int64_t)w * B + b) * G + g] = make_float2((float)(a / n), (float)(q / n));
}

// dx = rstd (gamma dv - A - xhat Bq); 4 channels per thread, 32-bit indices in the image
__global__ void __launch_bounds__(kT) gn_bwd_apply_kernel(const float* __restrict__ dout,
                                                          const float* __restrict__ mask,
                                                          const float* __restrict__ x, int64_t s_x, int P, int C,
                                                          int G, const float2* __restrict__ stats,
                                                          const float2* __restrict__ coef,
                                                          const float* __restrict__ Wc, int64_t sW, int64_t g_off,
                                                          const int32_t* __restrict__ active,
                                                          float* __restrict__ dx) {
  const int w = blockIdx.y;
  if (active && !active[w]) return;
  const int B = gridDim.z, b = blockIdx.z, Cg = C / G;
  const float* gam = Wc + (int64_t)w * sW + g_off;
  const int64_t base = (int64_t)w * s_x + (int64_t)b * P * C;
  const float2* st = stats + ((int64_t)w * B + b) * G;
  const float2* cf = coef + ((int64_t)w * B + b) * G;
  const float4* dv4 = reinterpret_cast<const float4*>(dout + base);
  const float4* mk4 = mask ? reinterpret_cast<const float4*>(mask + base) : nullptr;
  const float4* x4 = reinterpret_cast<const float4*>(x + base);
  float4* o4 = reinterpret_cast<float4*>(dx + base);
  const int n4 = P * C / 4;
  for (int i = blockIdx.x * kT + threadIdx.x; i < n4; i += gridDim.x * kT) {
    const int c = (4 * i) & (C - 1);
    const float4 dd = dv4[i], xx = x4[i];
    const float4 mm = mk4 ? mk4[i] : make_float4(1.f, 1.f, 1.f, 1.f);
    const float dva[4] = {dd.x, dd.y, dd.z, dd.w}, xa[4] = {xx.x, xx.y, xx.z, xx.w};
    const float ma[4] = {mm.x, mm.y, mm.z, mm.w};
    float o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int g = (c + e) / Cg;
      const float dv = ma[e] > 0.f ? dva[e] : 0.f;
      const float2 ms = st[g], ab = cf[g];
      const float xh = (xa[e] - ms.x) * ms.y;
      o[e] = ms.y * (gam[c + e] * dv - ab.x - xh * ab.y);
    }
    o4[i] = make_float4(o[0], o[1], o[2], o[3]);
  }
}

// dgamma / dbeta into G: warp per channel, lanes over (image, chunk) in order
__global__ void gn_param_grad_kernel(const double2* __restrict__ part, int B, int C, int nch,
                                     const int32_t* __restrict__ active, float* __restrict__ Gr, int64_t sW,
                                     int64_t g_off, int64_t b_off) {
  const int w = blockIdx.y;
  if (active && !active[w]) return;
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (c >= C) return;
  double a = 0.0, q = 0.0;
  for (int e = lane; e < B * nch; e += 32) {
    const double2 v = part[((int64_t)w * B * nch + e) * C + c];
    a += v.x;
    q += v.y;
  }
  a = warp_sum(a);
  q = warp_sum(q);
  if (lane == 0) {
    Gr[(int64_t)w * sW + g_off + c] = (float)q;
    Gr[(int64_t)w * sW + b_off + c] = (float)a;
  }
}

// ----------------------------------------------------------------- maxpool
// 3x3 / 2, pad 1; ties to the first maximum in row-major window order.  Grid (x, slot,
// image); 4 channels per thread (C % 4 == 0), 32-bit indices within the image.
__global__ void maxpool_kernel(const float* __restrict__ a, int64_t s_a, int C, int hin, int hout,
                               const int32_t* __restrict__ active, float* __restrict__ y, int64_t s_y,
                               uint8_t* __restrict__ arg) {
  const int w = blockIdx.y, b = blockIdx.z;
  if (active && !active[w]) return;
  const int c4n = C / 4, n = hout * hout * c4n;
  const float* ab = a + (int64_t)w * s_a + (int64_t)b * hin * hin * C;
  float* yb = y + (int64_t)w * s_y + (int64_t)b * hout * hout * C;
  uint8_t* gb = arg + (int64_t)w * s_y + (int64_t)b * hout * hout * C;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int c = (i % c4n) * 4, pix = i / c4n;
    const int oy = pix / hout, ox = pix - oy * hout;
    float best[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    int bi[4] = {0, 0, 0, 0};
    for (int ky = 0; ky < 3; ++ky) {
      const int iy = oy * 2 - 1 + ky;
      if (iy < 0 || iy >= hin) continue;
      for (int kx = 0; kx < 3; ++kx) {
        const int ix = ox * 2 - 1 + kx;
        if (ix < 0 || ix >= hin) continue;
        const float4 v = *reinterpret_cast<const float4*>(ab + (iy * hin + ix) * C + c);
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (vv[e] > best[e]) {
            best[e] = vv[e];
            bi[e] = ky * 3 + kx;
          }
      }
    }
    *reinterpret_cast<float4*>(yb + pix * C + c) = make_float4(best[0], best[1], best[2], best[3]);
    *reinterpret_cast<uchar4*>(gb + pix * C + c) = make_uchar4(bi[0], bi[1], bi[2], bi[3]);
  }
}

__global__ void maxpool_bwd_kernel(const float* __restrict__ dy, const uint8_t* __restrict__ arg, int64_t s_y, int C,
                                   int hin, int hout, const int32_t* __restrict__ active, float* __restrict__ da,
                                   int64_t s_a) {
  const int w = blockIdx.y, b = blockIdx.z;
  if (active && !active[w]) return;
  const int c4n = C / 4, n = hin * hin * c4n;
  const float* db = dy + (int64_t)w * s_y + (int64_t)b * hout * hout * C;
  const uint8_t* gb = arg + (int64_t)w * s_y + (int64_t)b * hout * hout * C;
  float* ob = da + (int64_t)w * s_a + (int64_t)b * hin * hin * C;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int c = (i % c4n) * 4, pix = i / c4n;
    const int y = pix / hin, x = pix - y * hin;
    float s[4] = {0.f, 0.f, 0.f, 0.f};
    // windows (oy, ox) with 2 oy - 1 <= y <= 2 oy + 1, in row-major order
    for (int oy = max(0, (y - 1) / 2); oy <= min(hout - 1, (y + 1) / 2); ++oy) {
      const int ky = y - (oy * 2 - 1);
      if (ky < 0 || ky > 2) continue;
      for (int ox = max(0, (x - 1) / 2); ox <= min(hout - 1, (x + 1) / 2); ++ox) {
        const int kx = x - (ox * 2 - 1);
        if (kx < 0 || kx > 2) continue;
        const int o = (oy * hout + ox) * C + c;
        const uchar4 g4 = *reinterpret_cast<const uchar4*>(gb + o);
        const float4 d4 = *reinterpret_cast<const float4*>(db + o);
        const int tap = ky * 3 + kx;
        if (g4.x == tap) s[0] += d4.x;
        if (g4.y == tap) s[1] += d4.y;
        if (g4.z == tap) s[2] += d4.z;
        if (g4.w == tap) s[3] += d4.w;
      }
    }
    *reinterpret_cast<float4*>(ob + pix * C + c) = make_float4(s[0], s[1], s[2], s[3]);
  }
}

// -------------------------------------------------------------------- head
// feat[w][b][c] = mean over the P pixels (fixed order)
__global__ void avgpool_kernel(const float* __restrict__ x, int64_t s_x, int B, int P, int C,
                               const int32_t* __restrict__ active, float* __restrict__ feat) {
  const int w = blockIdx.y;
  if (active && !active[w]) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * C) return;
  const int b = i / C, c = i - b * C;
  const float* p = x + (int64_t)w * s_x + (int64_t)b * P * C + c;
  float s = 0.f;
  for (int q = 0; q < P; ++q) s += p[(int64_t)q * C];
  feat[((int64_t)w * B + b) * C + c] = s / (float)P;
}

__global__ void avgpool_bwd_kernel(const float* __restrict__ dfeat, int B, int P, int C,
                                   const int32_t* __restrict__ active, float* __restrict__ dx, int64_t s_x) {
  const int w = blockIdx.y;
  if (active && !active[w]) return;
  const int64_t total = (int64_t)B * P * C;
  const float inv = 1.0f / (float)P;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const int b = (int)(i / ((int64_t)P * C));
    dx[(int64_t)w * s_x + i] = dfeat[((int64_t)w * B + b) * C + c] * inv;
  }
}

__device__ __forceinline__ float bce(float z, float y) { return fmaxf(z, 0.f) - z * y + log1pf(expf(-fabsf(z))); }

// One warp per image slot.  train: dz = (sigmoid(z) - y) / (K cnt) for the batch's
// images, 0 past it; row_loss / row_hit (nullable) = per-image mean BCE and the
// exact-match flag (0 past the batch).  cnt = nvalid[w] (train) or every slot.
__global__ void bce_kernel(const float* __restrict__ z, const float* __restrict__ lab, int B, int K,
                           const int32_t* __restrict__ nvalid, const int64_t* __restrict__ rows, float* __restrict__ dz,
                           float* __restrict__ row_loss, int32_t* __restrict__ row_hit, int total_slots) {
  const int slot = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (slot >= total_slots) return;
  const int w = slot / B, b = slot - w * B;
  const bool live = nvalid ? b < nvalid[w] : rows[slot] >= 0;
  const float inv = nvalid && nvalid[w] > 0 ? 1.0f / ((float)K * (float)nvalid[w]) : 0.f;
  float ls = 0.f;
  int miss = 0;
  for (int k = lane; k < K; k += 32) {
    const float zz = z[(int64_t)slot * K + k], yy = lab[(int64_t)slot * K + k];
    if (live) {
      ls += bce(zz, yy);
      miss |= (zz > 0.f) != (yy > 0.5f);
    }
    if (dz) dz[(int64_t)slot * K + k] = live ? (1.0f / (1.0f + expf(-zz)) - yy) * inv : 0.f;
  }
  ls = warp_sum(ls);
  miss = __any_sync(0xffffffffu, miss);
  if (row_loss && lane == 0) {
    row_loss[slot] = live ? ls / (float)K : 0.f;
    row_hit[slot] = live && !miss;
  }
}

__global__ void colsum_kernel(const float* __restrict__ dz, int B, int K, const int32_t* __restrict__ active,
                              float* __restrict__ Gr, int64_t sW, int64_t off) {
  const int w = blockIdx.y;
  if (active && !active[w]) return;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  float s = 0.f;
  for (int b = 0; b < B; ++b) s += dz[((int64_t)w * B + b) * K + k];
  Gr[(int64_t)w * sW + off + k] = s;
}

// per-client eval sums over a chunk of images in client-major order
__global__ void eval_accum_kernel(const float* __restrict__ row_loss, const int32_t* __restrict__ row_hit,
                                  const int64_t* __restrict__ img_off, const int32_t* __restrict__ num_rows, int C,
                                  int64_t g0, int cnt, double* __restrict__ loss, int32_t* __restrict__ correct,
                                  int skip) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int64_t nc = num_rows[c] - min(skip, num_rows[c]);
  const int64_t lo = img_off[c] > g0 ? img_off[c] : g0;
  const int64_t hi = img_off[c] + nc < g0 + cnt ? img_off[c] + nc : g0 + cnt;
  if (lo >= hi) return;
  double s = 0.0;
  int k = 0;
  for (int64_t g = lo; g < hi; ++g) {
    s += (double)row_loss[g - g0];
    k += row_hit[g - g0];
  }
  loss[c] += s;
  correct[c] += k;
}

// the first local step's batch (at theta_t) added to its client's evaluation sums
__global__ void step0_eval_kernel(const float* __restrict__ row_loss, const int32_t* __restrict__ row_hit,
                                  const int32_t* __restrict__ nvalid, const int32_t* __restrict__ ord, int c0, int W,
                                  int B, double* __restrict__ loss, int32_t* __restrict__ correct) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= W || nvalid[w] == 0) return;
  double s = 0.0;
  int k = 0;
  for (int b = 0; b < nvalid[w]; ++b) {
    s += (double)row_loss[(int64_t)w * B + b];
    k += row_hit[(int64_t)w * B + b];
  }
  const int c = ord[c0 + w];
  loss[c] += s;
  correct[c] += k;
}

// ------------------------------------------------------------ wave steps
__global__ void init_wave_kernel(const float* __restrict__ theta_t, int64_t D, float* __restrict__ Wc, int64_t sW,
                                 float* __restrict__ Dl, int64_t ldD, const int32_t* __restrict__ ord, int c0,
                                 int32_t* __restrict__ bad) {
  const int w = blockIdx.y, c = ord[c0 + w];
  if (blockIdx.x == 0 && threadIdx.x == 0) bad[c] = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < D; i += (int64_t)gridDim.x * blockDim.x) {
    Wc[(int64_t)w * sW + i] = theta_t[i];
    Dl[(int64_t)c * ldD + i] = 0.f;
  }
}

// theta <- theta - lr * (g + mu * (theta - theta_t) + control); delta accumulates the step
__global__ void sgd_kernel(float* __restrict__ Wc, const float* __restrict__ Gr, int64_t sW, float* __restrict__ Dl,
                           int64_t ldD, const float* __restrict__ control, int64_t ldc, int64_t D, float lr, float mu,
                           const int32_t* __restrict__ nvalid, const int32_t* __restrict__ ord, int c0) {
  const int w = blockIdx.y;
  if (nvalid[w] == 0) return;
  const int c = ord[c0 + w];
  float* W = Wc + (int64_t)w * sW;
  const float* g = Gr + (int64_t)w * sW;
  float* dl = Dl + (int64_t)c * ldD;
  const float* ct = control ? control + (int64_t)c * ldc : nullptr;
  // 16-byte path over the aligned prefix when every row is 16-byte aligned (scalar tail); the
  // same arithmetic per element
  const auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  int64_t i0 = 0;  // first element of the scalar tail
  if (a16(W) && a16(g) && a16(dl) && (!ct || a16(ct))) {
    i0 = D & ~(int64_t)3;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (D >> 2); i += (int64_t)gridDim.x * blockDim.x) {
      const float4 gv = reinterpret_cast<const float4*>(g)[i];
      float4 dv = reinterpret_cast<float4*>(dl)[i];
      float4 wv = reinterpret_cast<float4*>(W)[i];
      const float4 cv = ct ? reinterpret_cast<const float4*>(ct)[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      const float gs[4] = {gv.x, gv.y, gv.z, gv.w}, cs[4] = {cv.x, cv.y, cv.z, cv.w};
      float* dp4 = &dv.x;
      float* wp4 = &wv.x;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float x = gs[e];
        if (mu != 0.f) x = fmaf(mu, -dp4[e], x);
        if (ct) x += cs[e];
        x *= lr;
        wp4[e] -= x;
        dp4[e] += x;
      }
      reinterpret_cast<float4*>(W)[i] = wv;
      reinterpret_cast<float4*>(dl)[i] = dv;
    }
  }
  for (int64_t i = i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < D; i += (int64_t)gridDim.x * blockDim.x) {
    float s = g[i];
    if (mu != 0.f) s = fmaf(mu, -dl[i], s);
    if (ct) s += ct[i];
    s *= lr;
    W[i] -= s;
    dl[i] += s;
  }
}

// bad[c] |= any non-finite entry of client c's delta (bad zeroed by init_wave_kernel)
__global__ void nonfinite_kernel(const float* __restrict__ Dl, int64_t ldD, int64_t D, const int32_t* __restrict__ ord,
                                 int c0, int32_t* __restrict__ bad) {
  const int c = ord[c0 + blockIdx.y];
  int b = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < D; i += (int64_t)gridDim.x * blockDim.x)
    b |= !isfinite(Dl[(int64_t)c * ldD + i]);
  b = __syncthreads_or(b);
  if (threadIdx.x == 0 && b) atomicOr(&bad[c], 1);
}

// per (slot, chunk) activity of a split-K launch
__global__ void expand_active_kernel(const int32_t* __restrict__ active, int W, int S, int32_t* __restrict__ out) {
  const int z = blockIdx.x * blockDim.x + threadIdx.x;
  if (z < W * S) out[z] = active ? (active[z / S] != 0) : 1;
}

// the S chunk partials of a split-K weight gradient summed in chunk order
__global__ void ksplit_reduce_kernel(const float* __restrict__ part, int S, int64_t n,
                                     const int32_t* __restrict__ active, float* __restrict__ out, int64_t s_out) {
  const int w = blockIdx.y;
  if (active && !active[w]) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float a = 0.f;
    for (int q = 0; q < S; ++q) a += part[((int64_t)w * S + q) * n + i];
    out[(int64_t)w * s_out + i] = a;
  }
}

// ord[rank] = client, ranks by num_rows descending, ties by client index (a stable sort)
__global__ void order_kernel(const int32_t* __restrict__ num_rows, int C, int32_t* __restrict__ ord) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int n = num_rows[c];
  int r = 0;
  for (int j = 0; j < C; ++j) {
    const int m = num_rows[j];
    r += m > n || (m == n && j < c);
  }
  ord[r] = c;
}

__global__ void ones_kernel(int32_t* p, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = 1;
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

struct BlockAct {
  float *t1, *u1, *t2, *td, *out;
  float2 *st1, *st2, *std_;
};

struct Work {
  int W, B;
  int64_t s_stem, s_pool, s_max, s_col;  // per-slot strides (floats)
  int64_t* rows;
  float* lab;
  int32_t *nvalid, *ones, *hit, *ord;
  int64_t* img_off;
  float *Wc, *G, *wperm, *gperm, *stem_in;
  float *c1, *a1, *m1;  // stem conv output, GN + ReLU, maxpool
  uint8_t* arg;
  float2* st0;
  BlockAct blk[8];
  float *feat, *logits, *dz, *dfeat, *rloss;
  float *col, *dcol, *gA, *gB, *gT, *gTd, *sc, *kpart;
  int32_t* act_split;
  double2* part;
  float2* coef;
};

inline int64_t max_col(const Net& n) {
  int64_t m = (int64_t)n.stem.pout() * n.stem.kp();
  for (const Block& b : n.blk) {
    m = std::max(m, (int64_t)b.c1.pout() * b.c1.kp());
    m = std::max(m, (int64_t)b.c2.pout() * b.c2.kp());
    if (b.has_ds) m = std::max(m, (int64_t)b.ds.pout() * b.ds.kp());
  }
  return m;
}
inline int64_t max_part(const Net& n) {  // partial-sum entries per image (backward: per channel)
  auto f = [](int P, int C) { return (int64_t)nchunks(P, C) * C; };
  int64_t m = f(n.stem.pout(), n.m.w);
  for (const Block& b : n.blk) m = std::max(m, f(b.c1.pout(), b.c1.co));
  return m;
}

inline Work carve(const Net& n, int W, int B, bool train, Buf& b) {
  const Dims& m = n.m;
  const int64_t sW = (n.D + 3) & ~int64_t(3);
  Work k;
  k.W = W;
  k.B = B;
  k.s_stem = (int64_t)B * n.stem.pout() * m.w;
  k.s_pool = (int64_t)B * n.hp * n.hp * m.w;
  k.s_max = k.s_stem;
  k.s_col = (int64_t)B * max_col(n);
  k.rows = b.take<int64_t>((size_t)W * B);
  k.lab = b.take<float>((size_t)W * B * m.K);
  k.nvalid = b.take<int32_t>(W);
  k.ones = b.take<int32_t>(W);
  k.hit = b.take<int32_t>((size_t)W * B);
  k.ord = b.take<int32_t>(65536);
  k.img_off = b.take<int64_t>(65536);
  k.Wc = train ? b.take<float>((size_t)W * sW) : nullptr;
  k.G = train ? b.take<float>((size_t)W * sW) : nullptr;
  k.wperm = b.take<float>((size_t)W * n.P);
  k.gperm = train ? b.take<float>((size_t)W * n.P) : nullptr;
  k.stem_in = b.take<float>((size_t)W * B * m.S * m.S * 3);
  k.c1 = b.take<float>((size_t)W * k.s_stem);
  k.a1 = b.take<float>((size_t)W * k.s_stem);
  k.m1 = b.take<float>((size_t)W * k.s_pool);
  k.arg = b.take<uint8_t>((size_t)W * k.s_pool);
  k.st0 = b.take<float2>((size_t)W * B * m.G);
  for (int i = 0; i < 8; ++i) {
    const Block& q = n.blk[i];
    const size_t e = (size_t)W * B * q.c1.pout() * q.c1.co;
    BlockAct& a = k.blk[i];
    a.t1 = b.take<float>(e);
    a.u1 = b.take<float>(e);
    a.t2 = b.take<float>(e);
    a.td = q.has_ds ? b.take<float>(e) : nullptr;
    a.out = b.take<float>(e);
    a.st1 = b.take<float2>((size_t)W * B * m.G);
    a.st2 = b.take<float2>((size_t)W * B * m.G);
    a.std_ = q.has_ds ? b.take<float2>((size_t)W * B * m.G) : nullptr;
  }
  const int F = 8 * m.w;
  k.feat = b.take<float>((size_t)W * B * F);
  k.logits = b.take<float>((size_t)W * B * m.K);
  k.dz = b.take<float>((size_t)W * B * m.K);
  k.dfeat = b.take<float>((size_t)W * B * F);
  k.rloss = b.take<float>((size_t)W * B);
  k.col = b.take<float>((size_t)W * k.s_col);
  int64_t kp_max = 0;  // split-K partials per slot
  for (int j = 0; j < n.nconv; ++j) {
    const Conv& v = n.convs[j];
    const int S = ksplit(B * v.pout());
    if (S > 1) kp_max = std::max(kp_max, (int64_t)S * v.kp() * v.co);
  }
  k.kpart = train && kp_max ? b.take<float>((size_t)W * kp_max) : nullptr;
  k.act_split = b.take<int32_t>((size_t)W * 16);
  k.sc = b.take<float>((size_t)W * k.s_pool);  // downsample-branch output (<= a pooled map)
  k.part = b.take<double2>((size_t)W * B * max_part(n));
  k.coef = b.take<float2>((size_t)W * B * m.G);
  if (train) {
    k.dcol = b.take<float>((size_t)W * k.s_col);
    k.gA = b.take<float>((size_t)W * k.s_max);
    k.gB = b.take<float>((size_t)W * k.s_max);
    k.gT = b.take<float>((size_t)W * k.s_max);
    k.gTd = b.take<float>((size_t)W * k.s_pool);
  } else {
    k.dcol = k.gA = k.gB = k.gT = k.gTd = nullptr;
  }
  return k;
}

inline unsigned grid_for(int64_t total, int64_t per_block = 256 * 8) {
  int64_t g = (total + per_block - 1) / per_block;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(g, 4096));
}

// ------------------------------------------------------------ layer steps
struct Ctx {
  const Net* n;
  const Work* k;
  const float* Wc;  // weights (wave rows, or the shared theta with sW = 0)
  int64_t sW;
  int W, B;
  const int32_t* active;
  const float* X;
  int64_t ldx;
  cudaStream_t s;
};

// per-slot stride of conv cv's im2col rows: compact (B * P_out * kp), so the rows of all
// slots form one uniformly strided array (the split-K weight gradient below relies on it)
inline int64_t col_stride(const Ctx& c, const Conv& cv) { return (int64_t)c.B * cv.pout() * cv.kp(); }

// im2col of conv cv over the NHWC source src (per-slot stride s_src)
int im2col(const Ctx& c, const Conv& cv, const float* src, int64_t s_src) {
  const Work& k = *c.k;
  const bool vec = cv.ci % 4 == 0;
  const int64_t rows = (int64_t)c.B * cv.pout();
  const dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((rows + kRows - 1) / kRows, 8192)), c.W);
  if (vec) FB_LAUNCH("rn_im2col_kernel", c.s, (im2col_kernel<true><<<grid, 256, 0, c.s>>>(
                                                  src, s_src, c.B, cv.ci, cv.hin, cv.k, cv.stride, cv.pad, cv.hout,
                                                  cv.kp(), c.active, k.col, col_stride(c, cv))));
  else FB_LAUNCH("rn_im2col_kernel", c.s, (im2col_kernel<false><<<grid, 256, 0, c.s>>>(
                                              src, s_src, c.B, cv.ci, cv.hin, cv.k, cv.stride, cv.pad, cv.hout,
                                              cv.kp(), c.active, k.col, col_stride(c, cv))));
  return launch_status("rn im2col");
}

inline ConvTable table(const Net& n) {
  ConvTable t{};
  t.n = n.nconv;
  for (int j = 0; j < n.nconv; ++j) {
    const Conv& v = n.convs[j];
    t.w_off[j] = v.w_off;
    t.p_off[j] = v.p_off;
    t.co[j] = v.co;
    t.ci[j] = v.ci;
    t.kk[j] = v.k * v.k;
    t.kp[j] = v.kp();
  }
  return t;
}

// the step's conv weights into O(HW)I rows (W slots, or one shared copy when sW == 0)
int permute_weights(const Ctx& c) {
  const Work& k = *c.k;
  const int slots = c.sW ? c.W : 1;
  FB_LAUNCH("rn_permute_kernel", c.s, (permute_kernel<<<dim3(64, slots, c.n->nconv), 256, 0, c.s>>>(
                                          table(*c.n), c.n->P, c.Wc, c.sW, k.wperm, c.n->P,
                                          c.sW ? c.active : nullptr, 1)));
  return launch_status("rn permute");
}

// y = conv(src) (per slot y stride s_y)
int conv_fwd(const Ctx& c, const Conv& cv, const float* src, int64_t s_src, float* y, int64_t s_y) {
  int st = im2col(c, cv, src, s_src);
  if (st) return st;
  const Work& k = *c.k;
  Gemm g = gemm_base();
  g.A = k.col; g.lda = cv.kp(); g.sA = col_stride(c, cv);
  g.B = k.wperm + cv.p_off; g.ldb = cv.kp(); g.sB = c.sW ? c.n->P : 0;
  g.C = y; g.ldc = cv.co; g.sC = s_y;
  g.M = c.B * cv.pout(); g.N = cv.co; g.K = cv.kp();
  g.active = c.active;
  return rn_gemm(false, true, g, c.W, c.s);
}

// GroupNorm statistics of x (P pixels x C channels per image)
int gn_stats(const Ctx& c, const float* x, int64_t s_x, int P, int C, float2* stats) {
  const Work& k = *c.k;
  const int G = c.n->m.G, nch = nchunks(P, C), chunk = std::max(1, kChunkElems / C);
  const dim3 grid(nch, c.B, c.W);
  if (C <= 256) FB_LAUNCH("rn_gn_stats_kernel", c.s, (gn_stats_kernel<1><<<grid, kT, 0, c.s>>>(
                                                         x, s_x, P, C, G, chunk, nch, c.active, k.part)));
  else FB_LAUNCH("rn_gn_stats_kernel", c.s, (gn_stats_kernel<2><<<grid, kT, 0, c.s>>>(
                                                x, s_x, P, C, G, chunk, nch, c.active, k.part)));
  const int warps = 8;
  FB_LAUNCH("rn_gn_finalize_kernel", c.s, (gn_finalize_kernel<<<dim3((c.B * G + warps - 1) / warps, c.W), 32 * warps,
                                                                  0, c.s>>>(k.part, c.B, G, nch,
                                                                            (double)P * (C / G), c.active, stats)));
  return launch_status("rn gn stats");
}

int gn_apply(const Ctx& c, const float* x, int64_t s_x, int P, int C, const float2* stats, const Norm& nm,
             const float* res, bool relu, float* y) {
  const int64_t n = (int64_t)P * C / 4;
  const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + kT * 4 - 1) / (kT * 4), 1024));
  FB_LAUNCH("rn_gn_apply_kernel", c.s, (gn_apply_kernel<<<dim3(gx, c.W, c.B), kT, 0, c.s>>>(
                                           x, s_x, P, C, c.n->m.G, stats, c.Wc, c.sW, nm.g_off, nm.b_off, res,
                                           relu ? 1 : 0, c.active, y)));
  return launch_status("rn gn apply");
}

int forward(const Ctx& c) {
  const Net& n = *c.n;
  const Work& k = *c.k;
  const int w = n.m.w;
  int st;
  const int Ps = n.stem.pout();
  if ((st = permute_weights(c))) return st;
  const int64_t s_in0 = (int64_t)c.B * n.m.S * n.m.S * 3;
  FB_LAUNCH("rn_stem_input_kernel", c.s, (stem_input_kernel<<<dim3(grid_for(s_in0), c.W), 256, 0, c.s>>>(
                                             c.X, c.ldx, k.rows, c.B, n.m.S, c.active, k.stem_in)));
  if ((st = conv_fwd(c, n.stem, k.stem_in, s_in0, k.c1, k.s_stem))) return st;
  if ((st = gn_stats(c, k.c1, k.s_stem, Ps, w, k.st0))) return st;
  if ((st = gn_apply(c, k.c1, k.s_stem, Ps, w, k.st0, n.n0, nullptr, true, k.a1))) return st;
  const unsigned gp = (unsigned)((n.hp * n.hp * (w / 4) + 255) / 256);
  FB_LAUNCH("rn_maxpool_kernel", c.s, (maxpool_kernel<<<dim3(gp, c.W, c.B), 256, 0, c.s>>>(
                                          k.a1, k.s_stem, w, n.hs, n.hp, c.active, k.m1, k.s_pool, k.arg)));
  const float* x = k.m1;
  int64_t s_x = k.s_pool;
  for (int i = 0; i < 8; ++i) {
    const Block& q = n.blk[i];
    const BlockAct& a = k.blk[i];
    const int P = q.c1.pout(), C = q.c1.co;
    const int64_t s_o = (int64_t)c.B * P * C;
    if ((st = conv_fwd(c, q.c1, x, s_x, a.t1, s_o))) return st;
    if ((st = gn_stats(c, a.t1, s_o, P, C, a.st1))) return st;
    if ((st = gn_apply(c, a.t1, s_o, P, C, a.st1, q.n1, nullptr, true, a.u1))) return st;
    if ((st = conv_fwd(c, q.c2, a.u1, s_o, a.t2, s_o))) return st;
    if ((st = gn_stats(c, a.t2, s_o, P, C, a.st2))) return st;
    const float* res = x;
    if (q.has_ds) {
      if ((st = conv_fwd(c, q.ds, x, s_x, a.td, s_o))) return st;
      if ((st = gn_stats(c, a.td, s_o, P, C, a.std_))) return st;
      if ((st = gn_apply(c, a.td, s_o, P, C, a.std_, q.nd, nullptr, false, k.sc))) return st;
      res = k.sc;  // (stride s_o: the sc buffer holds one block output per slot)
    }
    if ((st = gn_apply(c, a.t2, s_o, P, C, a.st2, q.n2, res, true, a.out))) return st;
    x = a.out;
    s_x = s_o;
  }
  const int F = 8 * w, P4 = n.blk[7].c2.pout();
  FB_LAUNCH("rn_avgpool_kernel", c.s, (avgpool_kernel<<<dim3((c.B * F + 255) / 256, c.W), 256, 0, c.s>>>(
                                          x, s_x, c.B, P4, F, c.active, k.feat)));
  Gemm g = gemm_base();  // logits = feat fc^T + b
  g.A = k.feat; g.lda = F; g.sA = (int64_t)c.B * F;
  g.B = c.Wc + n.fc_w; g.ldb = F; g.sB = c.sW;
  g.C = k.logits; g.ldc = n.m.K; g.sC = (int64_t)c.B * n.m.K;
  g.M = c.B; g.N = n.m.K; g.K = F;
  g.bias = c.Wc + n.fc_b; g.sBias = c.sW;
  g.active = c.active;
  return rn_gemm(false, true, g, c.W, c.s);
}

// GroupNorm backward for y = norm(x) [+ res] [ReLU]: dv = dy * (mask > 0) (mask = the
// block output, or nullptr), dx = norm backward; dgamma / dbeta into G.
int gn_backward(const Ctx& c, const float* dy, const float* mask, const float* x, int64_t s_x, int P, int C,
                const float2* stats, const Norm& nm, float* dx) {
  const Work& k = *c.k;
  const int G = c.n->m.G, nch = nchunks(P, C), chunk = std::max(1, kChunkElems / C);
  const dim3 grid(nch, c.B, c.W);
  if (C <= 256) FB_LAUNCH("rn_gn_bwd_stats_kernel", c.s, (gn_bwd_stats_kernel<1><<<grid, kT, 0, c.s>>>(
                                                             dy, mask, x, s_x, P, C, G, stats, chunk, nch, c.active,
                                                             k.part)));
  else FB_LAUNCH("rn_gn_bwd_stats_kernel", c.s, (gn_bwd_stats_kernel<2><<<grid, kT, 0, c.s>>>(
                                                    dy, mask, x, s_x, P, C, G, stats, chunk, nch, c.active, k.part)));
  const int warps = 8;
  FB_LAUNCH("rn_gn_bwd_finalize_kernel", c.s,
            (gn_bwd_finalize_kernel<<<dim3((c.B * G + warps - 1) / warps, c.W), 32 * warps, 0, c.s>>>(
                k.part, c.B, C, G, nch, (double)P * (C / G), c.Wc, c.sW, nm.g_off, c.active, k.coef)));
  FB_LAUNCH("rn_gn_param_grad_kernel", c.s,
            (gn_param_grad_kernel<<<dim3((C + warps - 1) / warps, c.W), 32 * warps, 0, c.s>>>(
                k.part, c.B, C, nch, c.active, k.G, c.sW, nm.g_off, nm.b_off)));
  const int64_t n = (int64_t)P * C / 4;
  const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + kT * 4 - 1) / (kT * 4), 1024));
  FB_LAUNCH("rn_gn_bwd_apply_kernel", c.s, (gn_bwd_apply_kernel<<<dim3(gx, c.W, c.B), kT, 0, c.s>>>(
                                               dy, mask, x, s_x, P, C, G, stats, k.coef, c.Wc, c.sW, nm.g_off,
                                               c.active, dx)));
  return launch_status("rn gn backward");
}

// conv backward: dWp into gperm (im2col recomputed), and (dx != nullptr) dx =
// col2im(dT Wp) [+ add * (mask > 0)] (accumulate: dx += ...)
int conv_backward(const Ctx& c, const Conv& cv, const float* src, int64_t s_src, const float* dT, int64_t s_T,
                  float* dx, int64_t s_dx, const float* add, const float* mask, bool accumulate) {
  const Work& k = *c.k;
  int st = im2col(c, cv, src, s_src);
  if (st) return st;
  Gemm g = gemm_base();  // dWp^T = col^T dT ([kp][co]: M = kp fills the 128-row tiles)
  const int rows = c.B * cv.pout(), S = ksplit(rows), Kc = rows / S;
  g.A = k.col; g.lda = cv.kp(); g.sA = (int64_t)Kc * cv.kp();  // batch z = slot * S + chunk
  g.B = dT; g.ldb = cv.co; g.sB = (int64_t)Kc * cv.co;
  g.M = cv.kp(); g.N = cv.co; g.K = Kc;
  if (S == 1) {
    g.C = k.gperm + cv.p_off; g.ldc = cv.co; g.sC = c.n->P;
    g.active = c.active;
    if ((st = rn_gemm(true, false, g, c.W, c.s))) return st;
  } else {
    FB_LAUNCH("rn_expand_active_kernel", c.s, (expand_active_kernel<<<(c.W * S + 255) / 256, 256, 0, c.s>>>(
                                                  c.active, c.W, S, k.act_split)));
    g.C = k.kpart; g.ldc = cv.co; g.sC = (int64_t)cv.kp() * cv.co;
    g.active = k.act_split;
    if ((st = rn_gemm(true, false, g, c.W * S, c.s))) return st;
    const int64_t n = (int64_t)cv.kp() * cv.co;
    FB_LAUNCH("rn_ksplit_reduce_kernel", c.s, (ksplit_reduce_kernel<<<dim3(grid_for(n), c.W), 256, 0, c.s>>>(
                                                  k.kpart, S, n, c.active, k.gperm + cv.p_off, c.n->P)));
  }
  if (!dx) return FB_OK;
  g = gemm_base();  // dcol = dT Wp
  g.A = dT; g.lda = cv.co; g.sA = s_T;
  g.B = k.wperm + cv.p_off; g.ldb = cv.kp(); g.sB = c.n->P;
  g.C = k.dcol; g.ldc = cv.kp(); g.sC = col_stride(c, cv);
  g.M = c.B * cv.pout(); g.N = cv.kk(); g.K = cv.co;
  g.active = c.active;
  if ((st = rn_gemm(false, false, g, c.W, c.s))) return st;
  const int64_t total = (int64_t)c.B * cv.pin() * (cv.ci / 4);
  const dim3 grid(grid_for(total), c.W);
#define FB_RN_COL2IM(K_, S_)                                                                                     \
  FB_LAUNCH("rn_col2im_kernel", c.s, (col2im_kernel<K_, S_><<<grid, 256, 0, c.s>>>(                              \
                                         k.dcol, col_stride(c, cv), cv.kp(), c.B, cv.ci, cv.hin, cv.pad, cv.hout, \
                                         c.active,                                                              \
                                         add, mask, accumulate ? 1 : 0, dx, s_dx)))
  if (cv.k == 3 && cv.stride == 1) FB_RN_COL2IM(3, 1);
  else if (cv.k == 3 && cv.stride == 2) FB_RN_COL2IM(3, 2);
  else if (cv.k == 1 && cv.stride == 2) FB_RN_COL2IM(1, 2);
  else FB_RN_COL2IM(1, 1);
#undef FB_RN_COL2IM
  return launch_status("rn conv backward");
}

// gradient of the step's mean loss into G (every entry written once)
int backward(const Ctx& c, bool eval_rows) {
  const Net& n = *c.n;
  const Work& k = *c.k;
  const int w = n.m.w, K = n.m.K, F = 8 * w;
  int st;
  const int slots = c.W * c.B;
  FB_LAUNCH("rn_bce_kernel", c.s, (bce_kernel<<<(slots + 7) / 8, 256, 0, c.s>>>(
                                      k.logits, k.lab, c.B, K, k.nvalid, k.rows, k.dz, eval_rows ? k.rloss : nullptr,
                                      eval_rows ? k.hit : nullptr, slots)));
  Gemm g = gemm_base();  // dfc = dz^T feat
  g.A = k.dz; g.lda = K; g.sA = (int64_t)c.B * K;
  g.B = k.feat; g.ldb = F; g.sB = (int64_t)c.B * F;
  g.C = k.G + n.fc_w; g.ldc = F; g.sC = c.sW;
  g.M = K; g.N = F; g.K = c.B;
  g.active = c.active;
  if ((st = rn_gemm(true, false, g, c.W, c.s))) return st;
  FB_LAUNCH("rn_colsum_kernel", c.s, (colsum_kernel<<<dim3((K + 31) / 32, c.W), 32, 0, c.s>>>(
                                         k.dz, c.B, K, c.active, k.G, c.sW, n.fc_b)));
  g = gemm_base();  // dfeat = dz fc
  g.A = k.dz; g.lda = K; g.sA = (int64_t)c.B * K;
  g.B = c.Wc + n.fc_w; g.ldb = F; g.sB = c.sW;
  g.C = k.dfeat; g.ldc = F; g.sC = (int64_t)c.B * F;
  g.M = c.B; g.N = F; g.K = K;
  g.active = c.active;
  if ((st = rn_gemm(false, false, g, c.W, c.s))) return st;
  const int P4 = n.blk[7].c2.pout();
  // dOut of the last block into gA (gradients of block outputs alternate gA / gB)
  float* dout = k.gA;
  float* dnext = k.gB;
  FB_LAUNCH("rn_avgpool_bwd_kernel", c.s, (avgpool_bwd_kernel<<<dim3(grid_for((int64_t)c.B * P4 * F), c.W), 256, 0,
                                                                c.s>>>(k.dfeat, c.B, P4, F, c.active, dout,
                                                                       (int64_t)c.B * P4 * F)));
  for (int i = 7; i >= 0; --i) {
    const Block& q = n.blk[i];
    const BlockAct& a = k.blk[i];
    const int P = q.c1.pout(), C = q.c1.co;
    const int64_t s_o = (int64_t)c.B * P * C;
    const float* xin = i > 0 ? k.blk[i - 1].out : k.m1;
    const int64_t s_in = i > 0 ? (int64_t)c.B * n.blk[i - 1].c1.pout() * n.blk[i - 1].c1.co : k.s_pool;
    // the gradient buffers (gA / gB / gT / gTd, W x s_max floats) take this block's
    // activation stride s_o; out = relu(gn2(t2) + sc): dv = dout * (out > 0)
    if ((st = gn_backward(c, dout, a.out, a.t2, s_o, P, C, a.st2, q.n2, k.gT))) return st;  // dt2
    if (q.has_ds) {
      if ((st = gn_backward(c, dout, a.out, a.td, s_o, P, C, a.std_, q.nd, k.gTd))) return st;  // dtd
    }
    // conv2: dW2, du1 = col2im(dt2 W2) into dnext (scratch, stride s_o)
    if ((st = conv_backward(c, q.c2, a.u1, s_o, k.gT, s_o, dnext, s_o, nullptr, nullptr, false))) return st;
    // gn1 with mask u1: dt1 into gT
    if ((st = gn_backward(c, dnext, a.u1, a.t1, s_o, P, C, a.st1, q.n1, k.gT))) return st;
    // conv1 backward into the block input's gradient (dnext, stride s_in):
    //   identity: dx = col2im(dt1 W1) + dv (dv = dout * (out > 0));  downsample: + col2im(dtd Wd)
    if ((st = conv_backward(c, q.c1, xin, s_in, k.gT, s_o, dnext, s_in, q.has_ds ? nullptr : dout,
                            q.has_ds ? nullptr : a.out, false)))
      return st;
    if (q.has_ds) {
      if ((st = conv_backward(c, q.ds, xin, s_in, k.gTd, s_o, dnext, s_in, nullptr, nullptr, true))) return st;
    }
    std::swap(dout, dnext);
  }
  // stem: dout = d(maxpool output) -> d a1 (into dnext, stem stride) -> GN (mask a1) -> conv dW
  const unsigned gb = (unsigned)((n.hs * n.hs * (w / 4) + 255) / 256);
  FB_LAUNCH("rn_maxpool_bwd_kernel", c.s, (maxpool_bwd_kernel<<<dim3(gb, c.W, c.B), 256, 0, c.s>>>(
                                              dout, k.arg, k.s_pool, w, n.hs, n.hp, c.active, dnext, k.s_stem)));
  if ((st = gn_backward(c, dnext, k.a1, k.c1, k.s_stem, n.stem.pout(), w, k.st0, n.n0, k.gT))) return st;
  if ((st = conv_backward(c, n.stem, k.stem_in, (int64_t)c.B * n.m.S * n.m.S * 3, k.gT, k.s_stem, nullptr, 0,
                          nullptr, nullptr, false)))
    return st;
  // the conv gradients back into G's OIHW rows
  FB_LAUNCH("rn_permute_kernel", c.s, (permute_kernel<<<dim3(64, c.W, n.nconv), 256, 0, c.s>>>(
                                          table(n), n.P, k.gperm, c.sW, k.G, n.P, c.active, 0)));
  return launch_status("rn backward");
}

}  // namespace rn
}  // namespace fb

extern "C" {

int64_t fb_resnet_num_params(const int32_t* dims) {
  if (!dims) return 0;
  const fb::rn::Dims m = fb::rn::parse(dims);
  if (!fb::rn::dims_ok(m)) return 0;
  return fb::rn::build(m).D;
}

int64_t fb_resnet_workspace_bytes(const int32_t* dims, int batch_size, int clients_per_wave) {
  if (!dims || batch_size < 1) return 0;
  const fb::rn::Dims m = fb::rn::parse(dims);
  if (!fb::rn::dims_ok(m)) return 0;
  const fb::rn::Net n = fb::rn::build(m);
  fb::rn::Buf a;
  fb::rn::carve(n, clients_per_wave > 0 ? clients_per_wave : 1, batch_size, true, a);
  return (int64_t)a.off + 256;
}

int fb_eval_resnet_f32(const float* theta, const int32_t* dims, const float* X, int64_t ldx, const int64_t* row_start,
                       const int32_t* num_rows, const int32_t* h_num_rows, int num_clients, double* loss_sum,
                       int32_t* correct, int batch_size, int groups, void* workspace, int64_t workspace_bytes,
                       const int32_t* perms, const int64_t* perm_off, int skip, void* stream) {
  FB_REQUIRE(dims != nullptr && h_num_rows != nullptr, "eval_resnet: null dims / host row counts");
  const fb::rn::Dims m = fb::rn::parse(dims);
  FB_UNSUPPORTED(fb::rn::dims_ok(m), "eval_resnet: unsupported shape (width a power of two in [4, 64], "
                                     "groups dividing it, image side in [32, 1024], classes <= 256)");
  FB_REQUIRE(ldx >= 3LL * m.S * m.S + m.K, "eval_resnet: row length below 3 S^2 + K");
  FB_REQUIRE(num_clients >= 0 && num_clients <= 65536 && batch_size >= 1 && groups >= 1, "eval_resnet: bad sizes");
  FB_REQUIRE(workspace_bytes >= fb_resnet_workspace_bytes(dims, batch_size, groups), "eval_resnet: workspace too small");
  FB_REQUIRE(!perms || (perm_off && skip >= 0), "eval_resnet: perms need perm_off and skip >= 0");
  cudaStream_t s = fb::as_stream(stream);
  if (num_clients == 0) return FB_OK;
  cudaMemsetAsync(loss_sum, 0, sizeof(double) * num_clients, s);
  cudaMemsetAsync(correct, 0, sizeof(int32_t) * num_clients, s);
  const fb::rn::Net n = fb::rn::build(m);
  fb::rn::Buf b;
  b.base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
  fb::rn::Work k = fb::rn::carve(n, groups, batch_size, true, b);
  const int W = groups, B = batch_size;
  const int sk = perms ? skip : 0;
  FB_LAUNCH("rn_ones_kernel", s, (fb::rn::ones_kernel<<<(W + 255) / 256, 256, 0, s>>>(k.ones, W)));
  FB_LAUNCH("rn_img_offsets_kernel", s, (fb::rn::img_offsets_kernel<<<1, 32, 0, s>>>(num_rows, num_clients,
                                                                                      k.img_off, sk)));
  int64_t total = 0;
  for (int c = 0; c < num_clients; ++c) total += h_num_rows[c] - (sk < h_num_rows[c] ? sk : h_num_rows[c]);
  const int chunk = W * B;
  const int64_t lab_off = 3LL * m.S * m.S;
  fb::rn::Ctx cx{&n, &k, theta, 0, W, B, k.ones, X, ldx, s};
  for (int64_t g0 = 0; g0 < total; g0 += chunk) {
    const int cnt = (int)(total - g0 < chunk ? total - g0 : chunk);
    FB_LAUNCH("rn_gather_eval_kernel", s, (fb::rn::gather_eval_kernel<<<(chunk + 127) / 128, 128, 0, s>>>(
                                              X, ldx, lab_off, m.K, row_start, k.img_off, num_clients, g0, cnt, chunk,
                                              perms, perm_off, num_rows, sk, k.rows, k.lab)));
    int st = fb::rn::forward(cx);
    if (st) return st;
    FB_LAUNCH("rn_bce_kernel", s, (fb::rn::bce_kernel<<<(chunk + 7) / 8, 256, 0, s>>>(
                                      k.logits, k.lab, B, m.K, nullptr, k.rows, nullptr, k.rloss, k.hit, chunk)));
    FB_LAUNCH("rn_eval_accum_kernel", s, (fb::rn::eval_accum_kernel<<<(num_clients + 127) / 128, 128, 0, s>>>(
                                             k.rloss, k.hit, k.img_off, num_rows, num_clients, g0, cnt, loss_sum,
                                             correct, sk)));
  }
  return fb::launch_status("eval_resnet");
}

int fb_local_sgd_resnet_f32(const float* theta_t, const int32_t* dims, const float* X, int64_t ldx,
                            const int64_t* row_start, const int32_t* num_rows, const int32_t* h_num_rows,
                            const int32_t* perms, const int64_t* perm_off, int num_clients, int epochs,
                            int batch_size, float lr, float prox_mu, const float* control, int64_t ld_control,
                            float* delta_out, int64_t ld_delta, int32_t* nonfinite, int clients_per_wave,
                            void* workspace, int64_t workspace_bytes, double* eval_loss, int32_t* eval_correct,
                            void* stream) {
  FB_REQUIRE(dims != nullptr && h_num_rows != nullptr, "local_sgd_resnet: null dims / host row counts");
  const fb::rn::Dims m = fb::rn::parse(dims);
  FB_UNSUPPORTED(fb::rn::dims_ok(m), "local_sgd_resnet: unsupported shape (width a power of two in [4, 64], "
                                     "groups dividing it, image side in [32, 1024], classes <= 256)");
  const fb::rn::Net n = fb::rn::build(m);
  const int64_t D = n.D;
  FB_REQUIRE(ldx >= 3LL * m.S * m.S + m.K, "local_sgd_resnet: row length below 3 S^2 + K");
  FB_REQUIRE(num_clients >= 0 && num_clients <= 65536 && epochs >= 0 && batch_size >= 1 && clients_per_wave >= 1 &&
                 ld_delta >= D,
             "local_sgd_resnet: bad sizes");
  FB_REQUIRE(workspace_bytes >= fb_resnet_workspace_bytes(dims, batch_size, clients_per_wave),
             "local_sgd_resnet: workspace too small");
  cudaStream_t s = fb::as_stream(stream);
  if (num_clients == 0) return FB_OK;
  fb::rn::Buf b;
  b.base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
  fb::rn::Work k = fb::rn::carve(n, clients_per_wave, batch_size, true, b);
  const int64_t sW = (D + 3) & ~int64_t(3);
  const int B = batch_size;
  // waves largest-first (stable): similar local step counts side by side
  std::vector<int32_t> ord(num_clients);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int c) { return h_num_rows[a] > h_num_rows[c]; });
  FB_LAUNCH("rn_order_kernel", s, (fb::rn::order_kernel<<<(num_clients + 255) / 256, 256, 0, s>>>(num_rows, num_clients,
                                                                                                  k.ord)));
  const int64_t lab_off = 3LL * m.S * m.S;
  for (int c0 = 0; c0 < num_clients; c0 += clients_per_wave) {
    const int W = num_clients - c0 < clients_per_wave ? num_clients - c0 : clients_per_wave;
    int max_steps = 0;
    for (int i = c0; i < c0 + W; ++i) {
      const int nr = h_num_rows[ord[i]];
      const int st = nr > 0 ? epochs * ((nr + B - 1) / B) : 0;
      max_steps = st > max_steps ? st : max_steps;
    }
    FB_LAUNCH("rn_init_wave_kernel", s, (fb::rn::init_wave_kernel<<<dim3(256, W), 256, 0, s>>>(
                                            theta_t, D, k.Wc, sW, delta_out, ld_delta, k.ord, c0, nonfinite)));
    fb::rn::Ctx cx{&n, &k, k.Wc, sW, W, B, k.nvalid, X, ldx, s};
    for (int step = 0; step < max_steps; ++step) {
      FB_LAUNCH("rn_gather_batch_kernel", s, (fb::rn::gather_batch_kernel<<<W, 128, 0, s>>>(
                                                 X, ldx, lab_off, m.K, row_start, num_rows, perms, perm_off, k.ord,
                                                 c0, epochs, B, step, k.rows, k.lab, k.nvalid)));
      int st = fb::rn::forward(cx);
      if (st) return st;
      const bool ev0 = step == 0 && eval_loss != nullptr;  // step 0 runs at theta_t: the batch's evaluation
      st = fb::rn::backward(cx, ev0);
      if (st) return st;
      if (ev0)
        FB_LAUNCH("rn_step0_eval_kernel", s, (fb::rn::step0_eval_kernel<<<(W + 127) / 128, 128, 0, s>>>(
                                                 k.rloss, k.hit, k.nvalid, k.ord, c0, W, B, eval_loss, eval_correct)));
      FB_LAUNCH("rn_sgd_kernel", s, (fb::rn::sgd_kernel<<<dim3(256, W), 256, 0, s>>>(
                                        k.Wc, k.G, sW, delta_out, ld_delta, control, ld_control, D, lr, prox_mu,
                                        k.nvalid, k.ord, c0)));
    }
    FB_LAUNCH("rn_nonfinite_kernel", s, (fb::rn::nonfinite_kernel<<<dim3(64, W), 256, 0, s>>>(
                                            delta_out, ld_delta, D, k.ord, c0, nonfinite)));
  }
  return fb::launch_status("local_sgd_resnet");
}

}  // extern "C"
