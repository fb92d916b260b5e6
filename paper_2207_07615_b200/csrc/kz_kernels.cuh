// kz_kernels.cuh -- sm_100a device code of PLSS Kaczmarz (section 7,
// L931-967): identity-column sketches S_k = [e_{i_1} .. e_{i_k}] in a given row order, so
// y_k = a_{i_k} (row i_k of A) and, with the orthogonal history P_{k-1}, Theta_{k-1} = diag(p_j^T p_j)
// (eq:pkKacz, L952-956):
//
//   d = Theta^{-1/2} P^T a_i,   gamma = r_{k-1}[i] / ((||a_i|| - ||d||)(||a_i|| + ||d||)),
//   p_k = gamma (a_i - P Theta^{-1} P^T a_i),   x_k = x_{k-1} + p_k,   r_k = r_{k-1} - A p_k
//
// P^T a_i is row i of the stored [A p_1 .. A p_{k-1}] (L961-966), so a step costs one pass over
// the n x hk history P (the GEMV, the HBM-bound part), one SpMV for A p_k and vector work:
//   (prep)      one CTA (the last CTA of the previous step's k_kz_resid; k_kz_prep after the
//               start): swap the dense copy of row i into `arow`, ||a_i||^2, g_j = AP[i][j],
//               w_j = g_j / theta_j, ||d||^2, gamma, skip flag (reading R20: row in the span of
//               the history, empty, or already satisfied)
//   k_kz_gemv   p_l = gamma (arow_l - sum_j P[j][l] w_j) (ascending j), p -> pk and P[:, hk],
//               x += p, per-CTA partials of theta = p^T p
//   (SpMV)      apk = A pk (the PLSS K1 segments in plain mode)
//   k_kz_resid  r -= apk, rho, AP[:, hk] = apk; last CTA: theta_hk, hk++ (reset at kmax, R21),
//               iteration record, stop test, then the next step's prep
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace plss {

constexpr int KZ_NT = 256;
constexpr double KZ_SKIP_REL = 1e-14;

struct KzState {
  int32_t hk;        // stored updates in the history
  int32_t skip;      // this step's row is skipped (p = 0)
  int32_t prev_row;  // row whose entries sit in arow (-1: none)
  int32_t skipped;   // rows skipped so far
  double gamma;
};

struct KzArgs {
  int64_t m, n;
  int32_t kmax;
  const int32_t* row_ptr;    // CSR of A (borrowed)
  const int32_t* col_idx;
  const double* val;
  const int32_t* rows;       // row schedule, one per step
  double* P;                 // n x kmax, column j at P + j n
  double* AP;                // m x kmax ROW-major: (A p_j)_l at AP[l kmax + j], so prep reads row i
                             // of [A p_1 .. A p_hk] contiguously
  double* theta;             // [kmax]
  double* w;                 // [kmax] Theta^{-1} P^T a_i
  double* arow;              // [n] dense copy of the current row, zero elsewhere
  double* pk;                // [n] the current update (input of the SpMV)
  double* apk;               // [m] A p_k
  double* r;
  double* x;
  double* part_th;           // [grid_gemv] theta partials
  double* part_rho;          // [2 grid_res] rho partials (publish_and_elect pairs)
  unsigned* counter;
  KzState* st;
  Ctl* ctl;
  double* rec;
  int32_t grid_gemv, grid_res;
  int32_t fused;             // rows <= KZ_FUSE_MAXROW: k_kz_resid computes (A p)_l itself
};
constexpr int KZ_FUSE_MAXROW = 32;

__device__ __forceinline__ bool kz_done(const KzArgs& a) { return a.ctl->done != 0; }

// Row preparation of the step that starts now (ctl->iters steps done), by a whole CTA: swap row
// i = rows[iters] into arow, ||a_i||^2, g_j = (A p_j)_i, w_j = g_j / theta_j, ||d||^2, gamma, skip.
// Runs in the last CTA of k_kz_resid of the previous step (r, A P, theta just written by other
// CTAs / this CTA: read through L2), and once from k_kz_prep after the start.
__device__ void kz_prep_body(const KzArgs& a, double (*sm)[MAXW]) {
  const int t = threadIdx.x;
  KzState* st = a.st;
  const int i = a.rows[a.ctl->iters];
  const int prev = st->prev_row;
  if (prev >= 0)
    for (int e = a.row_ptr[prev] + t; e < a.row_ptr[prev + 1]; e += KZ_NT) a.arow[a.col_idx[e]] = 0.0;
  __syncthreads();
  double aa = 0.0, dd = 0.0;
  for (int e = a.row_ptr[i] + t; e < a.row_ptr[i + 1]; e += KZ_NT) {
    const double v = a.val[e];
    a.arow[a.col_idx[e]] = v;
    aa = __dadd_rn(aa, __dmul_rn(v, v));
  }
  const int hk = st->hk;
  const double* apr = a.AP + (int64_t)i * a.kmax;
  for (int j = t; j < hk; j += KZ_NT) {
    const double g = __ldcg(apr + j);
    const double th = __ldcg(a.theta + j);
    a.w[j] = __ddiv_rn(g, th);
    dd = __dadd_rn(dd, __ddiv_rn(__dmul_rn(g, g), th));
  }
  block_sum2(aa, dd, sm);
  if (t == 0) {
    const double na = __dsqrt_rn(aa), nd = __dsqrt_rn(dd);
    const double denom = __dmul_rn(__dadd_rn(na, -nd), __dadd_rn(na, nd));
    const double ri = __ldcg(a.r + i);
    const bool skip = aa == 0.0 || denom <= KZ_SKIP_REL * aa || ri == 0.0;   // reading R20
    st->skip = skip ? 1 : 0;
    st->gamma = skip ? 0.0 : __ddiv_rn(ri, denom);
    st->prev_row = i;
    if (skip) st->skipped += 1;
  }
}

__global__ void __launch_bounds__(KZ_NT) k_kz_prep(KzArgs a) {
  if (kz_done(a) || a.ctl->iters >= a.ctl->maxit) return;
  __shared__ double sm[2][MAXW];
  kz_prep_body(a, sm);
}

// p = gamma (arow - P w). A CTA takes tiles of KZ_TL consecutive l (grid-stride); its KZ_JS thread
// groups each sum a contiguous quarter of the history columns j (ascending, 8 loads in flight per
// thread), and the quarters are added in order (((q0 + q1) + q2) + q3): a fixed order, with four
// times the loads in flight of one thread per l.
constexpr int KZ_TL = 64;                 // l per tile
constexpr int KZ_JS = KZ_NT / KZ_TL;      // history splits
__global__ void __launch_bounds__(KZ_NT) k_kz_gemv(KzArgs a) {
  if (kz_done(a)) return;
  __shared__ double sm[2][MAXW];
  __shared__ double part[KZ_JS][KZ_TL];
  const KzState* st = a.st;
  const int hk = st->hk, skip = st->skip;
  const double gamma = st->gamma;
  const int tl = threadIdx.x % KZ_TL, js = threadIdx.x / KZ_TL;
  const int j0 = (int)((int64_t)hk * js / KZ_JS), j1 = (int)((int64_t)hk * (js + 1) / KZ_JS);
  double* Pnew = a.P + (int64_t)hk * a.n;
  double th = 0.0, zero = 0.0;
  if (((a.n & 1) | ((reinterpret_cast<uintptr_t>(a.P) | reinterpret_cast<uintptr_t>(a.arow) |
                      reinterpret_cast<uintptr_t>(a.pk) | reinterpret_cast<uintptr_t>(a.x)) & 15)) == 0) {
    // even n, aligned P: a thread takes rows (l, l + 1) of a 2 KZ_TL-row tile with 16-byte loads
    // (8 columns x 16 B in flight); each row's sum keeps its ascending-j order
    __shared__ double2 part2[KZ_JS][KZ_TL];
    for (int64_t l0 = (int64_t)blockIdx.x * 2 * KZ_TL; l0 < a.n; l0 += (int64_t)gridDim.x * 2 * KZ_TL) {
      const int64_t l = l0 + 2 * tl;
      double2 t = make_double2(0.0, 0.0);
      if (l < a.n) {
        int j = j0;
        for (; j + 8 <= j1; j += 8) {
          double2 pv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) pv[u] = __ldg(reinterpret_cast<const double2*>(a.P + (int64_t)(j + u) * a.n + l));
          double wv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) wv[u] = __ldg(a.w + j + u);
          asm volatile("" ::: "memory");           // all 8 row-pair loads issue before the first use
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const double wj = wv[u];
            t.x = __dadd_rn(t.x, __dmul_rn(pv[u].x, wj));
            t.y = __dadd_rn(t.y, __dmul_rn(pv[u].y, wj));
          }
        }
        for (; j < j1; ++j) {
          const double2 pv = __ldg(reinterpret_cast<const double2*>(a.P + (int64_t)j * a.n + l));
          const double wj = __ldg(a.w + j);
          t.x = __dadd_rn(t.x, __dmul_rn(pv.x, wj));
          t.y = __dadd_rn(t.y, __dmul_rn(pv.y, wj));
        }
      }
      part2[js][tl] = t;
      __syncthreads();
      if (js == 0 && l < a.n) {
        double2 tt = part2[0][tl];
#pragma unroll
        for (int q = 1; q < KZ_JS; ++q) { tt.x = __dadd_rn(tt.x, part2[q][tl].x); tt.y = __dadd_rn(tt.y, part2[q][tl].y); }
        const double2 ar = *reinterpret_cast<const double2*>(a.arow + l);
        double2 p2v;
        p2v.x = skip ? 0.0 : __dmul_rn(gamma, __dadd_rn(ar.x, -tt.x));
        p2v.y = skip ? 0.0 : __dmul_rn(gamma, __dadd_rn(ar.y, -tt.y));
        *reinterpret_cast<double2*>(a.pk + l) = p2v;
        if (!skip) {
          *reinterpret_cast<double2*>(Pnew + l) = p2v;
          double2 xx = *reinterpret_cast<const double2*>(a.x + l);
          xx.x = __dadd_rn(xx.x, p2v.x);
          xx.y = __dadd_rn(xx.y, p2v.y);
          *reinterpret_cast<double2*>(a.x + l) = xx;
        }
        th = __dadd_rn(th, __dmul_rn(p2v.x, p2v.x));
        th = __dadd_rn(th, __dmul_rn(p2v.y, p2v.y));
      }
      __syncthreads();
    }
    block_sum2(th, zero, sm);
    if (threadIdx.x == 0) a.part_th[blockIdx.x] = th;
    return;
  }
  for (int64_t l0 = (int64_t)blockIdx.x * KZ_TL; l0 < a.n; l0 += (int64_t)gridDim.x * KZ_TL) {
    const int64_t l = l0 + tl;
    double t = 0.0;
    if (l < a.n) {
      const double* col = a.P + l;
      int j = j0;
      for (; j + 8 <= j1; j += 8) {
        double pv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) pv[u] = __ldg(col + (int64_t)(j + u) * a.n);
#pragma unroll
        for (int u = 0; u < 8; ++u) t = __dadd_rn(t, __dmul_rn(pv[u], __ldg(a.w + j + u)));
      }
      for (; j < j1; ++j) t = __dadd_rn(t, __dmul_rn(__ldg(col + (int64_t)j * a.n), __ldg(a.w + j)));
    }
    part[js][tl] = t;
    __syncthreads();
    if (js == 0 && l < a.n) {
      double tt = part[0][tl];
#pragma unroll
      for (int q = 1; q < KZ_JS; ++q) tt = __dadd_rn(tt, part[q][tl]);
      const double p = skip ? 0.0 : __dmul_rn(gamma, __dadd_rn(a.arow[l], -tt));
      a.pk[l] = p;
      if (!skip) {
        Pnew[l] = p;
        a.x[l] = __dadd_rn(a.x[l], p);
      }
      th = __dadd_rn(th, __dmul_rn(p, p));
    }
    __syncthreads();
  }
  block_sum2(th, zero, sm);
  if (threadIdx.x == 0) a.part_th[blockIdx.x] = th;
}

// FUSED: (A p)_l is this thread's own sequential ascending sum over row l (rows of <= KZ_FUSE_MAXROW
// entries; bitwise the plain SpMV's value), replacing the separate SpMV launch and its apk pass
template <bool FUSED>
__global__ void __launch_bounds__(KZ_NT) k_kz_resid(KzArgs a) {
  if (kz_done(a)) return;
  __shared__ double sm[2][MAXW];
  const KzState* st = a.st;
  const int hk = st->hk, skip = st->skip;
  const int64_t per = (a.m + gridDim.x - 1) / gridDim.x;
  const int64_t l0 = (int64_t)blockIdx.x * per, l1 = min(a.m, l0 + per);
  double* APnew = a.AP + hk;
  double rho = 0.0, zero = 0.0;
  for (int64_t l = l0 + threadIdx.x; l < l1; l += KZ_NT) {
    double q;
    if (FUSED) {
      q = 0.0;
      const int e1 = a.row_ptr[l + 1];
      for (int e = a.row_ptr[l]; e < e1; ++e) q = __dadd_rn(q, __dmul_rn(a.val[e], __ldg(a.pk + a.col_idx[e])));
    } else {
      q = a.apk[l];
    }
    const double rl = __dadd_rn(a.r[l], -q);
    a.r[l] = rl;
    if (!skip) APnew[l * a.kmax] = q;
    rho = __dadd_rn(rho, __dmul_rn(rl, rl));
  }
  if (!publish_and_elect(rho, zero, a.part_rho, a.part_rho, gridDim.x, a.counter, sm)) return;
  const double rho_t = rho;                          // valid in thread 0
  double thv = 0.0, z2 = 0.0;                        // theta = sum of the GEMV partials (fixed order)
  for (int g = threadIdx.x; g < a.grid_gemv; g += KZ_NT) thv = __dadd_rn(thv, __ldcg(a.part_th + g));
  block_sum2(thv, z2, sm);
  __shared__ int s_next;
  if (threadIdx.x == 0) {
    KzState* ws = a.st;
    Ctl* c = a.ctl;
    if (!skip) {
      a.theta[hk] = thv;
      ws->hk = (hk + 1 == a.kmax) ? 0 : hk + 1;        // reading R21: history reset at kmax
    }
    const int k = c->iters + 1;
    c->iters = k;
    const double h = __ddiv_rn(__dsqrt_rn(rho_t), c->nbd);
    double* rk = a.rec + (size_t)k * REC;
    rk[0] = h;
    rk[1] = rho_t;
    rk[2] = (double)skip;
    rk[3] = ws->gamma;
    rk[4] = thv;
    rk[5] = (double)ws->hk;
    c->rho = rho_t;
    if (rho_t == 0.0 || h <= c->tol) { c->done = 1; c->outcome = OUT_CONVERGED; }
    s_next = !c->done && k < c->maxit;
  }
  __syncthreads();
  if (s_next) kz_prep_body(a, sm);                  // the next step's row, with this whole CTA
}

}  // namespace plss
