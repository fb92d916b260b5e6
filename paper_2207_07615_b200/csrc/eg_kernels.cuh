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
//   k_eg_gemvT  partials of Y^T y and y^T y: CTA b stages tiles of y in shared memory, thread j
//               walks column j of its row range (ascending l)
//   k_eg_tri    one CTA: fixed-order sums of the partials, u = R^T g, u ./= delta, t_hat = R u,
//               delta, coefficient, skip (reading R22), append t_hat to R and 1/delta to D,
//               iteration counter
//   k_eg_gemv   p = coef (y - Y t_hat) (history split in 4, fixed-order combination), x += p,
//               append y to Y
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace plss {

constexpr int EG_NT = 256;
constexpr int EG_TILE = 2048;            // y rows per shared-memory tile (gemvT)
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
};

struct EgArgs {
  int64_t m, n;
  int32_t kmax, mode;
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
  double* gv;                 // [kmax] g, then u
  double* th;                 // [kmax] t_hat of this step
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

// partials of g_j = Y[:, j]^T y (j < hk) and y^T y over CTA b's contiguous row range
__global__ void __launch_bounds__(EG_NT) k_eg_gemvT(EgArgs a) {
  if (eg_done(a)) return;
  __shared__ double ys[EG_TILE];
  __shared__ double sm[2][MAXW];
  const int hk = a.st->hk;
  const int64_t per = (a.n + gridDim.x - 1) / gridDim.x;
  const int64_t l0 = (int64_t)blockIdx.x * per, l1 = min(a.n, l0 + per);
  double* out = a.part + (size_t)blockIdx.x * (a.kmax + 1);
  double yy = 0.0, z = 0.0;
  for (int64_t l = l0 + threadIdx.x; l < l1; l += EG_NT) {
    const double v = a.y[l];
    yy = __dadd_rn(yy, __dmul_rn(v, v));
  }
  block_sum2(yy, z, sm);
  if (threadIdx.x == 0) out[a.kmax] = yy;
  for (int jb = 0; jb < hk; jb += EG_NT) {
    const int j = jb + threadIdx.x;
    double acc = 0.0;
    for (int64_t t0 = l0; t0 < l1; t0 += EG_TILE) {
      const int cnt = (int)min((int64_t)EG_TILE, l1 - t0);
      __syncthreads();
      for (int e = threadIdx.x; e < cnt; e += EG_NT) ys[e] = a.y[t0 + e];
      __syncthreads();
      if (j < hk) {
        const double* col = a.Y + (int64_t)j * a.n + t0;
        int e = 0;
        for (; e + 8 <= cnt; e += 8) {
          double yv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) yv[u] = __ldg(col + e + u);
#pragma unroll
          for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, __dmul_rn(yv[u], ys[e + u]));
        }
        for (; e < cnt; ++e) acc = __dadd_rn(acc, __dmul_rn(__ldg(col + e), ys[e]));
      }
    }
    if (j < hk) out[j] = acc;
  }
}

__global__ void __launch_bounds__(EG_NT) k_eg_tri(EgArgs a) {
  if (eg_done(a)) return;
  __shared__ double sm[2][MAXW];
  __shared__ double s_yy, s_rs;
  EgState* st = a.st;
  const int hk = st->hk, K = a.kmax, t = threadIdx.x, lane = t & 31;
  // g_j and y^T y: one warp per entry, lane-strided over the CTA partials, fixed butterfly
  for (int e = t >> 5; e <= hk; e += EG_NT / 32) {
    const int col = e < hk ? e : K;
    double s = 0.0;
    for (int g = lane; g < a.grid_t; g += 32) s = __dadd_rn(s, a.part[(size_t)g * (K + 1) + col]);
    s = warp_sum(s);
    if (lane == 0) { if (e < hk) a.gv[e] = s; else s_yy = s; }
  }
  if (t == 0) {
    double rs;
    if (a.mode == EG_RESIDUAL) rs = a.ctl->rho;                    // r^T r of the last K1
    else if (a.mode == EG_IDENTITY) rs = a.r[st->cur_row];
    else { rs = 0.0; for (int g = 0; g < a.grid_s; ++g) rs = __dadd_rn(rs, a.part_rs[g]); }
    s_rs = rs;
  }
  __syncthreads();
  // u = R^T g: u_j = sum_{i<j} R[i][j] g_i - g_j, then u_j /= delta_j (stored in th)
  for (int j = t; j < hk; j += EG_NT) {
    const double* Rc = a.R + (size_t)j * K;
    double u = 0.0;
    for (int i = 0; i < j; ++i) u = __dadd_rn(u, __dmul_rn(Rc[i], a.gv[i]));
    a.th[j] = __dmul_rn(__dadd_rn(u, -a.gv[j]), a.dinv[j]);
  }
  __syncthreads();
  // t_hat = R u: t_hat_i = sum_{j>i} R[i][j] u_j - u_i; delta partial g_i t_hat_i
  double gt = 0.0, z = 0.0;
  for (int i = t; i < hk; i += EG_NT) {
    double v = 0.0;
    for (int j = i + 1; j < hk; ++j) v = __dadd_rn(v, __dmul_rn(a.R[(size_t)j * K + i], a.th[j]));
    const double ti = __dadd_rn(v, -a.th[i]);
    a.R[(size_t)hk * K + i] = ti;              // next column of R (valid only if not skipped)
    gt = __dadd_rn(gt, __dmul_rn(a.gv[i], ti));
  }
  block_sum2(gt, z, sm);
  __syncthreads();
  for (int i = t; i < hk; i += EG_NT) a.th[i] = a.R[(size_t)hk * K + i];
  if (t == 0) {
    const double yy = s_yy, rs = s_rs;
    const double delta = __dadd_rn(yy, -gt);
    const bool skip = yy == 0.0 || delta <= EG_SKIP_REL * yy || rs == 0.0;   // reading R22
    st->skip = skip ? 1 : 0;
    st->coef = skip ? 0.0 : __ddiv_rn(rs, delta);
    st->hk_use = hk;
    if (!skip) {
      a.dinv[hk] = __ddiv_rn(1.0, delta);
      st->hk = (hk + 1 == K) ? 0 : hk + 1;     // reading R21 / R22: history reset at kmax
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
}

// p = coef (y - Y t_hat): tiles of 64 l, 4 groups each summing a quarter of the history columns
__global__ void __launch_bounds__(EG_NT) k_eg_gemv(EgArgs a) {
  if (eg_done(a)) return;
  constexpr int TL = 64, JS = EG_NT / TL;
  __shared__ double part[JS][TL];
  const EgState* st = a.st;
  const int hk = st->hk_use, skip = st->skip;
  const double coef = st->coef;
  const int tl = threadIdx.x % TL, js = threadIdx.x / TL;
  const int j0 = (int)((int64_t)hk * js / JS), j1 = (int)((int64_t)hk * (js + 1) / JS);
  double* Ynew = a.Y + (int64_t)hk * a.n;
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
        for (int u = 0; u < 8; ++u) t = __dadd_rn(t, __dmul_rn(pv[u], __ldg(a.th + j + u)));
      }
      for (; j < j1; ++j) t = __dadd_rn(t, __dmul_rn(__ldg(col + (int64_t)j * a.n), __ldg(a.th + j)));
    }
    part[js][tl] = t;
    __syncthreads();
    if (js == 0 && l < a.n) {
      double tt = part[0][tl];
#pragma unroll
      for (int q = 1; q < JS; ++q) tt = __dadd_rn(tt, part[q][tl]);
      const double yl = a.y[l];
      const double pl = skip ? 0.0 : __dmul_rn(coef, __dadd_rn(yl, -tt));
      a.p[l] = pl;
      if (!skip) {
        Ynew[l] = yl;
        a.x[l] = __dadd_rn(a.x[l], pl);
      }
    }
    __syncthreads();
  }
}

}  // namespace plss
