// eg_kernels.cuh -- sm_100a device code of the growing-sketch engine with the triangular
// factorization (section 2.4, Thm 2.1 and Cor 2.2, L284-441):
// for a sketch column s_k (residual r_{k-1}, identity e_{rows[k-1]} or a binary32 Gaussian column),
// y_k = A^T s_k, and with the stored Y (n x hk), R = [t_1 .. t_hk] (t_j = [t_hat_j; -1; 0]),
// D = diag(1/delta_j):
//
//   g = Y^T y,  t_hat = R D R^T g (two triangular products),  delta = y^T y - g^T t_hat,
//   p = (s^T r / delta) (y - Y t_hat)  (Cor 2.2, no solves),  append y, t_hat, 1/delta
//
// Kernels per step (plus the sketch step, see plss.cu, and PLSS K1 for r <- r - A p, rho, stop):
//   k_eg_row    identity sketch: one CTA swaps row i into the dense y (y_k = a_i), s^T r = r[i]
//   k_eg_gauss  Gaussian sketch: s_i = binary32 normal (randomized projection's generator, r = 1),
//               partials of s^T r; y = A^T s follows by the K2 segments
//   k_eg_gemvT  partials of Y^T y and y^T y: 2D grid (4096-row ranges x 32-column groups), a warp
//               per column, lanes over the rows (coalesced 256-byte reads of Y, y from L1), fixed
//               butterfly per column
//   k_eg_red    fixed-order sums of the partials (a warp per entry, many CTAs): g, y^T y, s^T r
//   k_eg_triu   u = D R^T g: a warp per column of R (coalesced), many CTAs
//   k_eg_trit   t_hat = R u: CTAs of 32 rows, 8 warps striding the columns (coalesced 256-byte
//               rows of R), fixed-order combination; delta partials; the last CTA: delta,
//               coefficient, skip (reading R22), append t_hat to R and 1/delta to D, iteration
//               counter
//   k_eg_gemv   p = coef (y - Y t_hat) (history split in 4, fixed-order combination), x += p,
//               append y to Y
//
// QR variant (section 2.3, eq:ykeqQR / eq:pkQR, L247-282), compact WY: Q_h = H_1 .. H_h = I - V T V^T
// (Householder H_j = I - tau_j v_j v_j^T, V n x h unit-trapezoidal, T h x h upper triangular):
//   a = V^T y (k_eg_gemvT / k_eg_red), b = T^T a (k_qr_b), w = Q_h^T y = y - V b (k_qr_w; its last
//   CTA forms the reflector of w[h:]: alpha = -sign(w_h) ||w[h:]||, v = w[h:] - alpha e_h,
//   tau = 2 / v^T v, r_hh = alpha), V[:, h] = v (k_qr_v), c = V^T v (gemvT / red),
//   T[:, h] = [-tau T c; tau] and z = T_{h+1} V_{h+1}^T e_h (k_qr_tri, one pass over T's rows),
//   q = e_h - V z, p = (s^T r / r_hh) q (k_eg_gemv<QR>)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace plss {

constexpr int EG_NT = 256;
#ifndef PLSS_EG_RT
#define PLSS_EG_RT 4096               // 2048: -1.6% engine step rate on C2 (scripts/gpu_egrt.sh)
#endif
constexpr int EG_RT = PLSS_EG_RT;        // rows per CTA of the Y^T y kernel (grid.x = row ranges)
constexpr int EG_RT_SMALL = 512;         // ... while few column groups are active (small history)
constexpr int EG_CT = 32;                // columns per CTA of the Y^T y kernel (grid.y = column groups)
constexpr double EG_SKIP_REL = 1e-14;

enum { EG_RESIDUAL = 0, EG_IDENTITY = 1, EG_GAUSSIAN = 2 };

struct EgState {
  int32_t hk;        // stored columns after this step's tri
  int32_t hk_use;    // history columns this step's gemv uses (= its append column)
  int32_t skip;
  int32_t prev_row;  // identity sketch: row sitting in y
  int32_t skipped;
  int32_t cur_row;
  double coef;
  double alpha, tau, vh;   // QR: r_hh, the new reflector's tau and its entry h
};

struct EgArgs {
  int64_t m, n;
  int32_t kmax, mode, factor;  // factor 0: triangular R D R^T, 1: Householder QR (compact WY)
  const int32_t* row_ptr;
  const int32_t* col_idx;
  const double* val;
  const int32_t* rows;
  uint64_t key;               // Gaussian sketch: mix64(seed)
  double* s;                  // [m] Gaussian sketch column
  double* y;                  // [n] y_k
  double* Y;                  // n x kmax, column-major
  double* R;                  // kmax x kmax, column-major (t_hat_j in column j, rows < j)
  double* dinv;               // [kmax] 1/delta_j
  double* gv;                 // [kmax + 2] g | y^T y | s^T r (Gaussian)
  double* th;                 // [kmax] t_hat of this step
  double* uv;                 // [kmax] u = D R^T g
  double* part_tri;           // [2 grid_tri] delta partial pairs (publish_and_elect)
  unsigned* counter;
  int32_t grid_tri;
  // QR variant: V lives in Y, T in R
  double* w;                  // [n] Q_h^T y, then v
  double* cv;                 // [kmax + 2] V^T v
  double* zv;                 // [kmax + 2] T_{h+1} V_{h+1}^T e_h
  double* part_w;             // [2 grid_g] sigma partial pairs
  unsigned* counter2;
  double* part;               // [grid_t][kmax + 1] partials of Y^T y | y^T y
  double* part_rs;            // [grid_s] partials of s^T r (Gaussian)
  double* p;
  double* x;
  const double* r;
  EgState* st;
  Ctl* ctl;
  double* rec;
  int32_t grid_t, grid_s, grid_g;
};

__device__ __forceinline__ bool eg_done(const EgArgs& a) { return a.ctl->done != 0; }

__global__ void __launch_bounds__(EG_NT) k_eg_row(EgArgs a) {
  if (eg_done(a)) return;
  const int t = threadIdx.x;
  EgState* st = a.st;
  const int i = a.rows[a.ctl->iters];
  const int prev = st->prev_row;
  if (prev >= 0)
    for (int e = a.row_ptr[prev] + t; e < a.row_ptr[prev + 1]; e += EG_NT) a.y[a.col_idx[e]] = 0.0;
  __syncthreads();
  for (int e = a.row_ptr[i] + t; e < a.row_ptr[i + 1]; e += EG_NT) a.y[a.col_idx[e]] = a.val[e];
  if (t == 0) { st->prev_row = i; st->cur_row = i; }
}

__global__ void __launch_bounds__(EG_NT) k_eg_gauss(EgArgs a) {
  if (eg_done(a)) return;
  __shared__ double sm[2][MAXW];
  const uint64_t k = (uint64_t)(a.ctl->iters + 1);
  double acc = 0.0, z = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * EG_NT + threadIdx.x; i < a.m; i += (int64_t)gridDim.x * EG_NT) {
    float z0, z1;
    rp_pair(a.key, (k << 32) + (uint64_t)i, 1.0, z0, z1);       // h = 1, q = 0: column 0
    const double si = (double)z0;
    a.s[i] = si;
    acc = __dadd_rn(acc, __dmul_rn(si, a.r[i]));
  }
  block_sum2(acc, z, sm);
  if (threadIdx.x == 0) a.part_rs[blockIdx.x] = acc;
}

// partials of g_j = Y[:, j]^T y (j < hk) and y^T y: CTA (x, y) covers rows [x RT, (x+1) RT) and
// columns [y CT, (y+1) CT); warp w takes columns w, w + 8, w + 16, w + 24 at once (8 independent
// loads per lane step), lanes stride the rows (64 per lane per column, amortizing the butterfly)
// Two instances run per step: RT = EG_RT_SMALL while ceil(n / EG_RT) * ceil(hk / EG_CT) CTAs would
// leave the GPU under-filled (small histories), RT = EG_RT otherwise; the other one exits at once.
__device__ __forceinline__ int eg_rt(const EgArgs& a, int hk) {
  const int64_t big = ((a.n + EG_RT - 1) / EG_RT) * (int64_t)((hk + EG_CT - 1) / EG_CT);
  return big >= 2 * 148 ? EG_RT : EG_RT_SMALL;
}
template <int SRC, int RT = EG_RT>      // SRC 0: y (Y^T y and y^T y), 1: w = v (QR: V^T v)
__global__ void __launch_bounds__(EG_NT) k_eg_gemvT(EgArgs a) {
  if (eg_done(a)) return;
  const int hk = a.st->hk;
  if (eg_rt(a, hk) != RT) return;
  const double* vec = SRC == 0 ? a.y : a.w;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = EG_NT / 32;
  if ((int64_t)blockIdx.x * RT >= a.n && !(blockIdx.x == 0)) return;
  const int64_t l0 = (int64_t)blockIdx.x * RT, l1 = min(a.n, l0 + RT);
  double* out = a.part + (size_t)blockIdx.x * (a.kmax + 1);
  const int jc0 = blockIdx.y * EG_CT;
  if (SRC == 0 && warp == 0 && blockIdx.y == 0) {
    double yy = 0.0;
    for (int64_t l = l0 + lane; l < l1; l += 32) {
      const double v = __ldg(vec + l);
      yy = __dadd_rn(yy, __dmul_rn(v, v));
    }
    yy = warp_sum(yy);
    if (lane == 0) out[a.kmax] = yy;
  }
  // columns j, j + NW, j + 2 NW, j + 3 NW at once, rows two per lane step: 8 independent loads
  const int jend = min(hk, jc0 + EG_CT);
  int j = jc0 + warp;
  if (((a.n & 1) | ((reinterpret_cast<uintptr_t>(vec) | reinterpret_cast<uintptr_t>(a.Y)) & 15)) == 0) {
    // even n, aligned: 16-byte loads of row pairs (2p, 2p + 1), 2 pairs per lane step (8 x 16 B
    // in flight per lane); per column the lane sums its pairs in order, then the fixed butterfly
    const double2* v2 = reinterpret_cast<const double2*>(vec);
    const int64_t p1 = l1 >> 1;
    for (; j + 3 * NW < jend; j += 4 * NW) {
      const double2* c[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) c[q] = reinterpret_cast<const double2*>(a.Y + (int64_t)(j + q * NW) * a.n);
      double sa[4] = {0.0, 0.0, 0.0, 0.0}, sb[4] = {0.0, 0.0, 0.0, 0.0};
      int64_t pp = (l0 >> 1) + lane;
      for (; pp + 32 < p1; pp += 64) {
        const double2 y0 = __ldg(v2 + pp), y1 = __ldg(v2 + pp + 32);
        double2 v0[4], v1[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) { v0[q] = __ldg(c[q] + pp); v1[q] = __ldg(c[q] + pp + 32); }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          sa[q] = __dadd_rn(__dadd_rn(sa[q], __dmul_rn(v0[q].x, y0.x)), __dmul_rn(v0[q].y, y0.y));
          sb[q] = __dadd_rn(__dadd_rn(sb[q], __dmul_rn(v1[q].x, y1.x)), __dmul_rn(v1[q].y, y1.y));
        }
      }
      if (pp < p1) {
        const double2 y0 = __ldg(v2 + pp);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 v0 = __ldg(c[q] + pp);
          sa[q] = __dadd_rn(__dadd_rn(sa[q], __dmul_rn(v0.x, y0.x)), __dmul_rn(v0.y, y0.y));
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double v = warp_sum(__dadd_rn(sa[q], sb[q]));
        if (lane == 0) out[j + q * NW] = v;
      }
    }
  }
  for (; j + 3 * NW < jend; j += 4 * NW) {
    const double* c[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) c[q] = a.Y + (int64_t)(j + q * NW) * a.n;
    double sa[4] = {0.0, 0.0, 0.0, 0.0}, sb[4] = {0.0, 0.0, 0.0, 0.0};
    int64_t l = l0 + lane;
    for (; l + 32 < l1; l += 64) {
      const double y0 = __ldg(vec + l), y1 = __ldg(vec + l + 32);
      double v0[4], v1[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) { v0[q] = __ldg(c[q] + l); v1[q] = __ldg(c[q] + l + 32); }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        sa[q] = __dadd_rn(sa[q], __dmul_rn(v0[q], y0));
        sb[q] = __dadd_rn(sb[q], __dmul_rn(v1[q], y1));
      }
    }
    if (l < l1) {
      const double y0 = __ldg(vec + l);
#pragma unroll
      for (int q = 0; q < 4; ++q) sa[q] = __dadd_rn(sa[q], __dmul_rn(__ldg(c[q] + l), y0));
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double v = warp_sum(__dadd_rn(sa[q], sb[q]));
      if (lane == 0) out[j + q * NW] = v;
    }
  }
  for (; j < jend; j += NW) {
    const double* c0 = a.Y + (int64_t)j * a.n;
    double s0 = 0.0;
    for (int64_t l = l0 + lane; l < l1; l += 32) s0 = __dadd_rn(s0, __dmul_rn(__ldg(c0 + l), __ldg(vec + l)));
    s0 = warp_sum(s0);
    if (lane == 0) out[j] = s0;
  }
}

// gv[e] = sum over the gemvT CTAs of part[.][e] for e < hk, gv[kmax] = y^T y, gv[kmax+1] = s^T r
// (Gaussian): one warp per entry, lane-strided partial sums in CTA order, fixed butterfly
template <int DST>                      // 0: gv (+ y^T y, s^T r), 1: cv (QR: V^T v only)
__global__ void __launch_bounds__(EG_NT) k_eg_red(EgArgs a) {
  if (eg_done(a)) return;
  const int hk = a.st->hk, K = a.kmax, lane = threadIdx.x & 31;
  const int e = blockIdx.x * (EG_NT / 32) + (threadIdx.x >> 5);
  if (e > hk + 1 || (DST == 1 && e >= hk)) return;
  double s = 0.0;
  if (e <= hk) {
    const int col = e < hk ? e : K;
    const int rt = eg_rt(a, DST == 1 ? hk : hk);
    const int nr = (int)((a.n + rt - 1) / rt);        // row ranges of the Y^T y instance that ran
    for (int g = lane; g < nr; g += 32) s = __dadd_rn(s, a.part[(size_t)g * (K + 1) + col]);
  } else if (a.mode == EG_GAUSSIAN) {
    for (int g = lane; g < a.grid_s; g += 32) s = __dadd_rn(s, a.part_rs[g]);
  }
  s = warp_sum(s);
  if (lane == 0) {
    if (DST == 1) a.cv[e] = s;
    else a.gv[e < hk ? e : (e == hk ? K : K + 1)] = s;
  }
}

// u_j = (sum_{i<j} R[i][j] g_i - g_j) / delta_j for j < hk: one warp per j
__global__ void __launch_bounds__(EG_NT) k_eg_triu(EgArgs a) {
  if (eg_done(a)) return;
  const int hk = a.st->hk, K = a.kmax, lane = threadIdx.x & 31;
  const int j = blockIdx.x * (EG_NT / 32) + (threadIdx.x >> 5);
  if (j >= hk) return;
  const double* Rc = a.R + (size_t)j * K;
  double s = 0.0;
  for (int i = lane; i < j; i += 32) s = __dadd_rn(s, __dmul_rn(Rc[i], a.gv[i]));
  s = warp_sum(s);
  if (lane == 0) a.uv[j] = __dmul_rn(__dadd_rn(s, -a.gv[j]), a.dinv[j]);
}

// t_hat_i = sum_{j>i} R[i][j] u_j - u_i for the CTA's 32 rows i; delta = y^T y - g^T t_hat
__global__ void __launch_bounds__(EG_NT) k_eg_trit(EgArgs a) {
  if (eg_done(a)) return;
  __shared__ double sm[2][MAXW];
  __shared__ double pt[EG_NT / 32][32];
  EgState* st = a.st;
  const int hk = st->hk, K = a.kmax, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = EG_NT / 32;
  const int i = blockIdx.x * 32 + lane;
  double acc = 0.0;
  if (blockIdx.x * 32 < hk) {
    for (int j = blockIdx.x * 32 + 1 + warp; j < hk; j += NW)
      if (j > i) acc = __dadd_rn(acc, __dmul_rn(a.R[(size_t)j * K + i], a.uv[j]));
  }
  pt[warp][lane] = acc;
  __syncthreads();
  double gt = 0.0, z = 0.0;
  if (warp == 0 && i < hk) {
    double t = pt[0][lane];
#pragma unroll
    for (int w = 1; w < NW; ++w) t = __dadd_rn(t, pt[w][lane]);
    t = __dadd_rn(t, -a.uv[i]);
    a.th[i] = t;
    a.R[(size_t)hk * K + i] = t;               // next column of R (kept only if not skipped)
    gt = __dmul_rn(a.gv[i], t);
  }
  if (!publish_and_elect(gt, z, a.part_tri, a.part_tri, gridDim.x, a.counter, sm)) return;
  if (threadIdx.x != 0) return;
  double rs;
  if (a.mode == EG_RESIDUAL) rs = a.ctl->rho;                      // r^T r of the last K1
  else if (a.mode == EG_IDENTITY) rs = __ldcg(a.r + st->cur_row);
  else rs = a.gv[K + 1];
  const double yy = a.gv[K];
  const double delta = __dadd_rn(yy, -gt);
  const bool skip = yy == 0.0 || delta <= EG_SKIP_REL * yy || rs == 0.0;     // reading R22
  st->skip = skip ? 1 : 0;
  st->coef = skip ? 0.0 : __ddiv_rn(rs, delta);
  st->hk_use = hk;
  if (!skip) {
    a.dinv[hk] = __ddiv_rn(1.0, delta);
    st->hk = (hk + 1 == K) ? 0 : hk + 1;       // reading R21 / R22: history reset at kmax
  } else {
    st->skipped += 1;
  }
  Ctl* c = a.ctl;
  const int k = c->iters + 1;
  c->iters = k;
  double* rk = a.rec + (size_t)k * REC;
  rk[2] = delta;
  rk[3] = (double)skip;
  rk[4] = rs;
  rk[5] = (double)st->hk;
}

// sum over history columns j in [j0, j1), ascending, of Y[j][l] w_j for the row pair (l, l + 1):
// 16-byte loads of 8 columns per batch (Y column-major with an even leading dimension n)
__device__ __forceinline__ double2 eg_pair_sum(const double* Y, int64_t n, const double* w, int j0, int j1,
                                               int64_t l) {
  double2 t = make_double2(0.0, 0.0);
  int j = j0;
  for (; j + 8 <= j1; j += 8) {
    double2 pv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) pv[u] = __ldg(reinterpret_cast<const double2*>(Y + (int64_t)(j + u) * n + l));
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double wj = __ldg(w + j + u);
      t.x = __dadd_rn(t.x, __dmul_rn(pv[u].x, wj));
      t.y = __dadd_rn(t.y, __dmul_rn(pv[u].y, wj));
    }
  }
  for (; j < j1; ++j) {
    const double2 pv = __ldg(reinterpret_cast<const double2*>(Y + (int64_t)j * n + l));
    const double wj = __ldg(w + j);
    t.x = __dadd_rn(t.x, __dmul_rn(pv.x, wj));
    t.y = __dadd_rn(t.y, __dmul_rn(pv.y, wj));
  }
  return t;
}
__device__ __forceinline__ bool eg_pairs_ok(const EgArgs& a) {
  return ((a.n & 1) | ((reinterpret_cast<uintptr_t>(a.Y) | reinterpret_cast<uintptr_t>(a.y) |
                        reinterpret_cast<uintptr_t>(a.p) | reinterpret_cast<uintptr_t>(a.x) |
                        reinterpret_cast<uintptr_t>(a.w)) & 15)) == 0;
}

// p = coef (y - Y t_hat): tiles of 64 l (128 l as row pairs with 16-byte loads when n is even),
// 4 groups each summing a quarter of the history columns, quarters added in order.
// QR: p = coef (e_h - V z) over the h + 1 columns of V_{h+1} (the new column is already in V).
template <int QR>
__global__ void __launch_bounds__(EG_NT) k_eg_gemv(EgArgs a) {
  if (eg_done(a)) return;
  constexpr int TL = 64, JS = EG_NT / TL;
  __shared__ double part[JS][TL];
  __shared__ double2 part2[JS][TL];
  const EgState* st = a.st;
  const int hu = st->hk_use, skip = st->skip;
  const int hk = QR ? hu + 1 : hu;
  const double* wt = QR ? a.zv : a.th;
  const double coef = st->coef;
  const int tl = threadIdx.x % TL, js = threadIdx.x / TL;
  const int j0 = (int)((int64_t)hk * js / JS), j1 = (int)((int64_t)hk * (js + 1) / JS);
  double* Ynew = a.Y + (int64_t)hu * a.n;
  if (eg_pairs_ok(a)) {
    for (int64_t l0 = (int64_t)blockIdx.x * 2 * TL; l0 < a.n; l0 += (int64_t)gridDim.x * 2 * TL) {
      const int64_t l = l0 + 2 * tl;
      part2[js][tl] = l < a.n ? eg_pair_sum(a.Y, a.n, wt, j0, j1, l) : make_double2(0.0, 0.0);
      __syncthreads();
      if (js == 0 && l < a.n) {
        double2 tt = part2[0][tl];
#pragma unroll
        for (int q = 1; q < JS; ++q) { tt.x = __dadd_rn(tt.x, part2[q][tl].x); tt.y = __dadd_rn(tt.y, part2[q][tl].y); }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t le = l + e;
          const double yl = QR ? (le == hu ? 1.0 : 0.0) : a.y[le];
          const double pl = skip ? 0.0 : __dmul_rn(coef, __dadd_rn(yl, e ? -tt.y : -tt.x));
          a.p[le] = pl;
          if (!skip) {
            if (!QR) Ynew[le] = yl;
            a.x[le] = __dadd_rn(a.x[le], pl);
          }
        }
      }
      __syncthreads();
    }
    return;
  }
  for (int64_t l0 = (int64_t)blockIdx.x * TL; l0 < a.n; l0 += (int64_t)gridDim.x * TL) {
    const int64_t l = l0 + tl;
    double t = 0.0;
    if (l < a.n) {
      const double* col = a.Y + l;
      int j = j0;
      for (; j + 8 <= j1; j += 8) {
        double pv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) pv[u] = __ldg(col + (int64_t)(j + u) * a.n);
#pragma unroll
        for (int u = 0; u < 8; ++u) t = __dadd_rn(t, __dmul_rn(pv[u], __ldg(wt + j + u)));
      }
      for (; j < j1; ++j) t = __dadd_rn(t, __dmul_rn(__ldg(col + (int64_t)j * a.n), __ldg(wt + j)));
    }
    part[js][tl] = t;
    __syncthreads();
    if (js == 0 && l < a.n) {
      double tt = part[0][tl];
#pragma unroll
      for (int q = 1; q < JS; ++q) tt = __dadd_rn(tt, part[q][tl]);
      const double yl = QR ? (l == hu ? 1.0 : 0.0) : a.y[l];
      const double pl = skip ? 0.0 : __dmul_rn(coef, __dadd_rn(yl, -tt));
      a.p[l] = pl;
      if (!skip) {
        if (!QR) Ynew[l] = yl;
        a.x[l] = __dadd_rn(a.x[l], pl);
      }
    }
    __syncthreads();
  }
}

// ---- QR variant ------------------------------------------------------------------------------
// b_j = sum_{i <= j} T[i][j] a_i (b = T^T a), one warp per column j of T
__global__ void __launch_bounds__(EG_NT) k_qr_b(EgArgs a) {
  if (eg_done(a)) return;
  const int hk = a.st->hk, K = a.kmax, lane = threadIdx.x & 31;
  const int j = blockIdx.x * (EG_NT / 32) + (threadIdx.x >> 5);
  if (j >= hk) return;
  const double* Tc = a.R + (size_t)j * K;
  double s = 0.0;
  for (int i = lane; i <= j; i += 32) s = __dadd_rn(s, __dmul_rn(Tc[i], a.gv[i]));
  s = warp_sum(s);
  if (lane == 0) a.uv[j] = s;
}

// w = y - V b (history split), sigma = ||w[h:]||^2; the last CTA forms the reflector
__global__ void __launch_bounds__(EG_NT) k_qr_w(EgArgs a) {
  if (eg_done(a)) return;
  constexpr int TL = 64, JS = EG_NT / TL;
  __shared__ double part[JS][TL];
  __shared__ double sm[2][MAXW];
  EgState* st = a.st;
  const int hk = st->hk;
  const int tl = threadIdx.x % TL, js = threadIdx.x / TL;
  const int j0 = (int)((int64_t)hk * js / JS), j1 = (int)((int64_t)hk * (js + 1) / JS);
  double sig = 0.0, z = 0.0;
  const bool pairs = eg_pairs_ok(a);
  __shared__ double2 part2[JS][TL];
  for (int64_t l0 = (int64_t)blockIdx.x * 2 * TL; pairs && l0 < a.n; l0 += (int64_t)gridDim.x * 2 * TL) {
    const int64_t l = l0 + 2 * tl;            // row pairs with 16-byte loads (n even)
    part2[js][tl] = l < a.n ? eg_pair_sum(a.Y, a.n, a.uv, j0, j1, l) : make_double2(0.0, 0.0);
    __syncthreads();
    if (js == 0 && l < a.n) {
      double2 tt = part2[0][tl];
#pragma unroll
      for (int q = 1; q < JS; ++q) { tt.x = __dadd_rn(tt.x, part2[q][tl].x); tt.y = __dadd_rn(tt.y, part2[q][tl].y); }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t le = l + e;
        const double wl = __dadd_rn(a.y[le], e ? -tt.y : -tt.x);
        a.w[le] = wl;
        if (le >= hk) sig = __dadd_rn(sig, __dmul_rn(wl, wl));
      }
    }
    __syncthreads();
  }
  for (int64_t l0 = (int64_t)blockIdx.x * TL; !pairs && l0 < a.n; l0 += (int64_t)gridDim.x * TL) {
    const int64_t l = l0 + tl;
    double t = 0.0;
    if (l < a.n) {
      const double* col = a.Y + l;
      int j = j0;
      for (; j + 8 <= j1; j += 8) {
        double pv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) pv[u] = __ldg(col + (int64_t)(j + u) * a.n);
#pragma unroll
        for (int u = 0; u < 8; ++u) t = __dadd_rn(t, __dmul_rn(pv[u], __ldg(a.uv + j + u)));
      }
      for (; j < j1; ++j) t = __dadd_rn(t, __dmul_rn(__ldg(col + (int64_t)j * a.n), __ldg(a.uv + j)));
    }
    part[js][tl] = t;
    __syncthreads();
    if (js == 0 && l < a.n) {
      double tt = part[0][tl];
#pragma unroll
      for (int q = 1; q < JS; ++q) tt = __dadd_rn(tt, part[q][tl]);
      const double wl = __dadd_rn(a.y[l], -tt);
      a.w[l] = wl;
      if (l >= hk) sig = __dadd_rn(sig, __dmul_rn(wl, wl));
    }
    __syncthreads();
  }
  if (!publish_and_elect(sig, z, a.part_w, a.part_w, gridDim.x, a.counter2, sm)) return;
  if (threadIdx.x != 0) return;
  double rs;
  if (a.mode == EG_RESIDUAL) rs = a.ctl->rho;
  else if (a.mode == EG_IDENTITY) rs = __ldcg(a.r + st->cur_row);
  else rs = a.gv[a.kmax + 1];
  const double yy = a.gv[a.kmax];
  const bool skip = yy == 0.0 || hk >= a.n || sig <= EG_SKIP_REL * yy || rs == 0.0;    // reading R22
  double alpha = 0.0, tau = 0.0, vh = 0.0;
  if (!skip) {
    const double wh = __ldcg(a.w + hk);
    alpha = wh >= 0.0 ? -__dsqrt_rn(sig) : __dsqrt_rn(sig);
    vh = __dadd_rn(wh, -alpha);
    const double vv = __dadd_rn(__dadd_rn(sig, -__dmul_rn(wh, wh)), __dmul_rn(vh, vh));
    tau = __ddiv_rn(2.0, vv);
  }
  st->skip = skip ? 1 : 0;
  st->alpha = alpha;
  st->tau = tau;
  st->vh = vh;
  st->coef = skip ? 0.0 : __ddiv_rn(rs, alpha);           // p = (s^T r / r_hh) q, r_hh = alpha
  a.rec[(size_t)(a.ctl->iters + 1) * REC + 4] = rs;
}

// v = [0 (l < h); vh (l = h); w_l (l > h)] into w and, unless skipped, into V[:, h]
__global__ void __launch_bounds__(EG_NT) k_qr_v(EgArgs a) {
  if (eg_done(a)) return;
  const EgState* st = a.st;
  const int hk = st->hk, skip = st->skip;
  const double vh = st->vh;
  double* Vn = a.Y + (int64_t)hk * a.n;
  for (int64_t l = (int64_t)blockIdx.x * EG_NT + threadIdx.x; l < a.n; l += (int64_t)gridDim.x * EG_NT) {
    const double v = l < hk ? 0.0 : (l == hk ? vh : a.w[l]);
    a.w[l] = v;
    if (!skip) Vn[l] = v;
  }
}

// t_i = -tau sum_{i <= j < h} T[i][j] c_j (the new column of T) and
// z_i = sum_{i <= j < h} T[i][j] g_j + t_i vh with g_j = V[h][j] (row h of V) for the CTA's 32 rows;
// the last CTA: z_h = tau vh, T[h][h] = tau, history size, iteration counter, record
__global__ void __launch_bounds__(EG_NT) k_qr_tri(EgArgs a) {
  if (eg_done(a)) return;
  __shared__ double sm[2][MAXW];
  __shared__ double pt[EG_NT / 32][32], pz[EG_NT / 32][32];
  EgState* st = a.st;
  const int hk = st->hk, K = a.kmax, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = EG_NT / 32;
  const int i = blockIdx.x * 32 + lane;
  const double tau = st->tau, vh = st->vh;
  double at = 0.0, az = 0.0;
  if (blockIdx.x * 32 < hk) {
    for (int j = blockIdx.x * 32 + warp; j < hk; j += NW) {
      if (j >= i) {
        const double tij = a.R[(size_t)j * K + i];
        at = __dadd_rn(at, __dmul_rn(tij, a.cv[j]));
        az = __dadd_rn(az, __dmul_rn(tij, __ldg(a.Y + (int64_t)j * a.n + hk)));
      }
    }
  }
  pt[warp][lane] = at;
  pz[warp][lane] = az;
  __syncthreads();
  if (warp == 0 && i < hk) {
    double t = pt[0][lane], zz = pz[0][lane];
#pragma unroll
    for (int w = 1; w < NW; ++w) { t = __dadd_rn(t, pt[w][lane]); zz = __dadd_rn(zz, pz[w][lane]); }
    const double ti = -__dmul_rn(tau, t);
    a.R[(size_t)hk * K + i] = ti;                        // new column of T (kept only if not skipped)
    a.zv[i] = __dadd_rn(zz, __dmul_rn(ti, vh));
  }
  double z0 = 0.0, z1 = 0.0;
  if (!publish_and_elect(z0, z1, a.part_tri, a.part_tri, gridDim.x, a.counter, sm)) return;
  if (threadIdx.x != 0) return;
  const int skip = st->skip;
  a.zv[hk] = __dmul_rn(tau, vh);
  st->hk_use = hk;
  if (!skip) {
    a.R[(size_t)hk * K + hk] = tau;
    st->hk = (hk + 1 == K) ? 0 : hk + 1;
  } else {
    st->skipped += 1;
  }
  Ctl* c = a.ctl;
  const int k = c->iters + 1;
  c->iters = k;
  double* rk = a.rec + (size_t)k * REC;
  rk[2] = __dmul_rn(st->alpha, st->alpha);            // r_hh^2 = delta_k
  rk[3] = (double)skip;
  rk[5] = (double)st->hk;
}

}  // namespace plss
