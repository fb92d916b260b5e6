// rp_kernels.cuh -- sm_100a device code of randomized projection ("Rand. Proj.", the paper's
// comparison method): eq:pkLong with W = I and a fresh
// random S_k in R^{m x r} every iteration (L171-176; Experiment I L985-991: standard normal, r = 10;
// Experiment III L1164-1170: sparse normal; Fig. 2: r = 10/20/40):
//
//   p_k = Y_k (Y_k^T Y_k)^+ S_k^T r_{k-1},  Y_k = A^T S_k,   x_k = x_{k-1} + p_k,  r_k = r_{k-1} - A p_k
//
// One iteration = five kernels here + K1 of the PLSS path (r <- r - A p, rho, stop test):
//   k_rp_gen    S_k (row-major m x r) from the counter-based generator of DESIGN.md reading R7,
//               fused with the per-CTA partials of v = S_k^T r_{k-1}
//   k_rp_spmm   Y_k = A^T S_k as a gather over the CSC copy: a group of G lanes per column, lane c
//               sums column c of Y sequentially in ascending row order (bitwise the oracle's
//               per-column sequential sums for equal S)
//   k_rp_gram   per-CTA partials of the upper triangle of Y_k^T Y_k (fixed order)
//   k_rp_solve  one CTA: sums the partials in CTA order, pivoted Cholesky of the r x r Gram
//               matrix truncated at its numerical rank, z = M^+-equivalent solve (reading R8),
//               iteration counter
//   k_rp_update p = Y z, x <- x + p
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace plss {

constexpr int RP_RMAX = 64;        // largest sketch size r
constexpr int RP_ATT = 64;         // polar-method attempts per pair (P(all rejected) ~ 1e-43)
constexpr int RP_NT = 256;
constexpr int RP_TILE = 4096;      // doubles of Y per shared-memory tile of the Gram kernel (32 KB)
constexpr int RP_PPT = (RP_RMAX * (RP_RMAX + 1) / 2 + RP_NT - 1) / RP_NT;   // Gram pairs per thread

// ---- counter-based sketch generator (reading R7; the oracle implements the same definition) ----
__device__ __forceinline__ uint64_t rp_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t rp_word(uint64_t key, uint64_t ctr) {
  return rp_mix64(key + (ctr + 1ull) * 0x9E3779B97F4A7C15ull);
}
__device__ __forceinline__ double rp_unit(uint64_t w) {       // 53-bit uniform in [0, 1), exact
  return __dmul_rn((double)(w >> 11), 0x1p-53);
}
// ln(s), s in (0, 1): frexp, m in [sqrt(1/2), sqrt(2)), f = (m-1)/(m+1),
// ln m = 2 f (1 + f^2/3 + ... + f^22/23) by Horner, ln s = e ln2 + ln m; every op correctly
// rounded, no contraction: bitwise the oracle's ln_unit.
__device__ __forceinline__ double rp_ln(double s) {
  int e;
  double mt = frexp(s, &e);
  if (mt < 0.7071067811865476) { mt = __dmul_rn(mt, 2.0); e -= 1; }
  const double f = __ddiv_rn(__dadd_rn(mt, -1.0), __dadd_rn(mt, 1.0));
  const double f2 = __dmul_rn(f, f);
  double t = 1.0 / 23.0;
  t = __dadd_rn(__dmul_rn(t, f2), 1.0 / 21.0);
  t = __dadd_rn(__dmul_rn(t, f2), 1.0 / 19.0);
  t = __dadd_rn(__dmul_rn(t, f2), 1.0 / 17.0);
  t = __dadd_rn(__dmul_rn(t, f2), 1.0 / 15.0);
  t = __dadd_rn(__dmul_rn(t, f2), 1.0 / 13.0);
  t = __dadd_rn(__dmul_rn(t, f2), 1.0 / 11.0);
  t = __dadd_rn(__dmul_rn(t, f2), 1.0 / 9.0);
  t = __dadd_rn(__dmul_rn(t, f2), 1.0 / 7.0);
  t = __dadd_rn(__dmul_rn(t, f2), 1.0 / 5.0);
  t = __dadd_rn(__dmul_rn(t, f2), 1.0 / 3.0);
  t = __dadd_rn(__dmul_rn(t, f2), 1.0);
  return __dadd_rn(__dmul_rn((double)e, 0.6931471805599453), __dmul_rn(__dmul_rn(2.0, f), t));
}
// the normal pair (S[i, 2q], S[i, 2q+1]) of pair counter `base` = ((k 2^32 + i) h + q)
__device__ __forceinline__ void rp_pair(uint64_t key, uint64_t base, double density, double& z0, double& z1) {
  z0 = 0.0;
  z1 = 0.0;
  for (int a = 0; a < RP_ATT; ++a) {
    const uint64_t c = (base * RP_ATT + (uint64_t)a) * 4ull;
    const double u = __dadd_rn(__dmul_rn(2.0, rp_unit(rp_word(key, c))), -1.0);
    const double v = __dadd_rn(__dmul_rn(2.0, rp_unit(rp_word(key, c + 1ull))), -1.0);
    const double s = __dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v));
    if (s > 0.0 && s < 1.0) {
      const double f = __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, rp_ln(s)), s));
      z0 = __dmul_rn(u, f);
      z1 = __dmul_rn(v, f);
      break;
    }
  }
  if (density < 1.0) {
    const uint64_t c = base * (uint64_t)(RP_ATT * 4);
    if (!(rp_unit(rp_word(key, c + 2ull)) < density)) z0 = 0.0;
    if (!(rp_unit(rp_word(key, c + 3ull)) < density)) z1 = 0.0;
  }
}

// Control shared with the PLSS path: the ctx's Ctl (iters, done, stop test via K1's tail_rho).
struct RpArgs {
  int64_t m, n;
  int32_t r, h;              // sketch size, pairs per row = ceil(r/2)
  uint64_t key;              // mix64(seed)
  double density;            // 1: dense normal S; < 1: each entry kept with this probability
  int64_t k_fixed;           // > 0: generate S_{k_fixed} (test entry point, no ctl)
  double* S;                 // m x r row-major
  double* Y;                 // n x r row-major
  const double* res;         // r_{k-1} (for v = S^T r), or NULL
  double* vpart;             // [grid_gen][r]
  double* mpart;             // [grid_gram][r(r+1)/2]
  double* z;                 // [RP_RMAX]
  double* p;                 // update (n)
  double* x;                 // iterate (n)
  const int32_t* col_ptr;    // CSC of A
  const int32_t* row_idx;
  const double* val_t;
  int32_t grid_gen, grid_gram;
  Ctl* ctl;
  double* rec;
};

__device__ __forceinline__ bool rp_done(const RpArgs& a) { return a.ctl != nullptr && a.ctl->done; }

// S_k and v partials. CTA b owns rows [b*per, (b+1)*per); thread t -> pair q = t % h of rows
// lr = t / h, lr + rpp, ... (rpp = 256 / h rows per pass): consecutive threads write consecutive
// doubles. v partial of column c: sum over the CTA's threads of that column in lr order.
__global__ void __launch_bounds__(RP_NT) k_rp_gen(RpArgs a) {
  if (rp_done(a)) return;
  __shared__ double red[2][RP_NT];
  const int h = a.h, r = a.r;
  const int rpp = RP_NT / h;
  const int t = threadIdx.x, lr = t / h, q = t % h;
  const uint64_t k = a.k_fixed > 0 ? (uint64_t)a.k_fixed : (uint64_t)(a.ctl->iters + 1);
  const int64_t per = (a.m + gridDim.x - 1) / gridDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * per, i1 = min(a.m, i0 + per);
  const int c0 = 2 * q;
  const bool has1 = c0 + 1 < r;
  double acc0 = 0.0, acc1 = 0.0;
  if (lr < rpp) {
    for (int64_t i = i0 + lr; i < i1; i += rpp) {
      double z0, z1;
      rp_pair(a.key, ((k << 32) + (uint64_t)i) * (uint64_t)h + (uint64_t)q, a.density, z0, z1);
      double* row = a.S + i * r;
      row[c0] = z0;
      if (has1) row[c0 + 1] = z1;
      if (a.res) {
        const double ri = a.res[i];
        acc0 = __dadd_rn(acc0, __dmul_rn(z0, ri));
        acc1 = __dadd_rn(acc1, __dmul_rn(z1, ri));
      }
    }
  }
  if (!a.res) return;
  red[0][t] = acc0;
  red[1][t] = acc1;
  __syncthreads();
  if (t < r) {
    const int qq = t >> 1, e = t & 1;
    double s = 0.0;
    for (int l = 0; l < rpp; ++l) s = __dadd_rn(s, red[e][l * h + qq]);
    a.vpart[(size_t)blockIdx.x * r + t] = s;
  }
}

// Y = A^T S: G lanes per column (G = pow2 >= r, <= 32), lane g sums columns g, g + G (CPL = 2
// for r > 32). Entries are taken 4 at a time (independent gathers in flight), added in order.
template <int G, int CPL>
__global__ void __launch_bounds__(RP_NT) k_rp_spmm(RpArgs a) {
  if (rp_done(a)) return;
  const int r = a.r;
  const int lane = threadIdx.x & 31;
  const int sub = lane / G, g = lane % G;
  constexpr int CPW = 32 / G;                       // columns per warp
  const int64_t warp = ((int64_t)blockIdx.x * RP_NT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * RP_NT) >> 5;
  for (int64_t j = warp * CPW + sub; j < a.n; j += nwarps * CPW) {
    const int b = __ldg(a.col_ptr + j), e = __ldg(a.col_ptr + j + 1);
    double acc[CPL];
#pragma unroll
    for (int u = 0; u < CPL; ++u) acc[u] = 0.0;
    int t = b;
    for (; t + 4 <= e; t += 4) {
      int ri[4];
      double vv[4];
#pragma unroll
      for (int w = 0; w < 4; ++w) { ri[w] = __ldg(a.row_idx + t + w); vv[w] = __ldg(a.val_t + t + w); }
      double sv[4][CPL];
#pragma unroll
      for (int w = 0; w < 4; ++w)
#pragma unroll
        for (int u = 0; u < CPL; ++u) {
          const int c = g + u * G;
          sv[w][u] = c < r ? __ldg(a.S + (int64_t)ri[w] * r + c) : 0.0;
        }
#pragma unroll
      for (int w = 0; w < 4; ++w)
#pragma unroll
        for (int u = 0; u < CPL; ++u) acc[u] = __dadd_rn(acc[u], __dmul_rn(vv[w], sv[w][u]));
    }
    for (; t < e; ++t) {
      const int ri = __ldg(a.row_idx + t);
      const double vv = __ldg(a.val_t + t);
#pragma unroll
      for (int u = 0; u < CPL; ++u) {
        const int c = g + u * G;
        const double sv = c < r ? __ldg(a.S + (int64_t)ri * r + c) : 0.0;
        acc[u] = __dadd_rn(acc[u], __dmul_rn(vv, sv));
      }
    }
#pragma unroll
    for (int u = 0; u < CPL; ++u) {
      const int c = g + u * G;
      if (c < r) a.Y[j * r + c] = acc[u];
    }
  }
}

// pair index -> (i, j), i <= j, row-major over the upper triangle
__device__ __forceinline__ void rp_pair_ij(int pidx, int r, int& i, int& j) {
  int base = 0;
  i = 0;
  while (pidx >= base + (r - i)) { base += r - i; ++i; }
  j = i + (pidx - base);
}

// Gram partials: CTA b owns rows [b*per, (b+1)*per) of Y, staged RP_TILE / r rows at a time in
// shared memory. np = r(r+1)/2 pairs; with np <= 128 the threads form ngrp = 256/np groups, group g
// summing rows g, g+ngrp, ... of each tile; the groups are then added in group order.
__global__ void __launch_bounds__(RP_NT) k_rp_gram(RpArgs a) {
  if (rp_done(a)) return;
  __shared__ double tile[RP_TILE];
  __shared__ double red[RP_NT];
  const int r = a.r, np = r * (r + 1) / 2, t = threadIdx.x;
  const int rows = RP_TILE / r;
  const int ngrp = np <= RP_NT / 2 ? RP_NT / np : 1;
  const int grp = ngrp > 1 ? t / np : 0;
  int pi[RP_PPT], pj[RP_PPT];
  double acc[RP_PPT];
#pragma unroll
  for (int u = 0; u < RP_PPT; ++u) {
    acc[u] = 0.0;
    const int pidx = ngrp > 1 ? t % np : t + u * RP_NT;
    pi[u] = pj[u] = -1;
    if ((ngrp > 1 ? (u == 0 && grp < ngrp) : pidx < np)) rp_pair_ij(pidx, r, pi[u], pj[u]);
  }
  const int64_t per = (a.n + gridDim.x - 1) / gridDim.x;
  const int64_t j0 = (int64_t)blockIdx.x * per, j1 = min(a.n, j0 + per);
  for (int64_t jb = j0; jb < j1; jb += rows) {
    const int nr = (int)min((int64_t)rows, j1 - jb);
    __syncthreads();
    for (int e = t; e < nr * r; e += RP_NT) tile[e] = a.Y[jb * r + e];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < RP_PPT; ++u) {
      if (pi[u] < 0) continue;
      for (int rr = grp; rr < nr; rr += ngrp)
        acc[u] = __dadd_rn(acc[u], __dmul_rn(tile[rr * r + pi[u]], tile[rr * r + pj[u]]));
    }
  }
  double* out = a.mpart + (size_t)blockIdx.x * np;
  if (ngrp > 1) {
    __syncthreads();
    red[t] = (grp < ngrp && t < ngrp * np) ? acc[0] : 0.0;
    __syncthreads();
    if (t < np) {
      double s = 0.0;
      for (int g = 0; g < ngrp; ++g) s = __dadd_rn(s, red[g * np + t]);
      out[t] = s;
    }
  } else {
#pragma unroll
    for (int u = 0; u < RP_PPT; ++u)
      if (t + u * RP_NT < np) out[t + u * RP_NT] = acc[u];
  }
}

// One CTA: M = sum of Gram partials, v = sum of v partials (CTA order), pivoted Cholesky
// M = P L L^T P^T stopped when the largest remaining pivot <= r eps max_j M_jj (numerical rank),
// z = P [L11^-T L11^-1 (P^T v)_1 ; 0]. For a consistent system v = Y^T e lies in range(M) and
// null(M) = null(Y), so Y z equals Y M^+ v (reading R8).
__global__ void __launch_bounds__(RP_NT) k_rp_solve(RpArgs a) {
  if (rp_done(a)) return;
  __shared__ double M[RP_RMAX][RP_RMAX + 1];
  __shared__ double v[RP_RMAX], w[RP_RMAX];
  __shared__ int perm[RP_RMAX];
  __shared__ int s_piv, s_rank;
  __shared__ double s_thr;
  const int r = a.r, np = r * (r + 1) / 2, t = threadIdx.x, lane = t & 31;
  // one warp per entry of M (upper triangle) / of v: lane-strided partial sums, fixed butterfly
  for (int e = t >> 5; e < np + r; e += RP_NT / 32) {
    double s = 0.0;
    if (e < np) {
      for (int g = lane; g < a.grid_gram; g += 32) s = __dadd_rn(s, a.mpart[(size_t)g * np + e]);
    } else {
      for (int g = lane; g < a.grid_gen; g += 32) s = __dadd_rn(s, a.vpart[(size_t)g * r + (e - np)]);
    }
    s = warp_sum(s);
    if (lane == 0) {
      if (e < np) {
        int i, j;
        rp_pair_ij(e, r, i, j);
        M[i][j] = s;
        M[j][i] = s;
      } else {
        v[e - np] = s;
      }
    }
  }
  if (t < r) perm[t] = t;
  __syncthreads();
  if (t == 0) {
    double dmax = 0.0;
    for (int i = 0; i < r; ++i) dmax = fmax(dmax, M[i][i]);
    s_thr = (double)r * 2.220446049250313e-16 * dmax;
    s_rank = r;
  }
  __syncthreads();
  for (int kk = 0; kk < r; ++kk) {
    if (t == 0) {
      int p = kk;
      for (int i = kk + 1; i < r; ++i) if (M[i][i] > M[p][p]) p = i;
      if (!(M[p][p] > s_thr)) { s_rank = kk; p = -1; }
      s_piv = p;
    }
    __syncthreads();
    const int p = s_piv;
    if (p < 0) break;
    if (p != kk) {                                   // symmetric swap kk <-> p
      for (int j = t; j < r; j += RP_NT) { const double q = M[kk][j]; M[kk][j] = M[p][j]; M[p][j] = q; }
      __syncthreads();
      for (int i = t; i < r; i += RP_NT) { const double q = M[i][kk]; M[i][kk] = M[i][p]; M[i][p] = q; }
      if (t == 0) { const int q = perm[kk]; perm[kk] = perm[p]; perm[p] = q; }
      __syncthreads();
    }
    const double l = __dsqrt_rn(M[kk][kk]);
    __syncthreads();
    if (t == 0) M[kk][kk] = l;
    for (int i = kk + 1 + t; i < r; i += RP_NT) M[i][kk] = __ddiv_rn(M[i][kk], l);
    __syncthreads();
    // trailing update of the WHOLE (symmetric) trailing block: a later symmetric pivot swap moves
    // entries across the diagonal, so both triangles must stay current
    const int rem = r - kk - 1;
    for (int e = t; e < rem * rem; e += RP_NT) {
      const int i = kk + 1 + e / rem, j = kk + 1 + e % rem;
      M[i][j] = __dadd_rn(M[i][j], -__dmul_rn(M[i][kk], M[j][kk]));
    }
    __syncthreads();
  }
  if (t == 0) {
    const int rk = s_rank;
    for (int i = 0; i < rk; ++i) {                  // L w = P^T v
      double s = v[perm[i]];
      for (int j = 0; j < i; ++j) s = __dadd_rn(s, -__dmul_rn(M[i][j], w[j]));
      w[i] = __ddiv_rn(s, M[i][i]);
    }
    for (int i = rk - 1; i >= 0; --i) {             // L^T z' = w
      double s = w[i];
      for (int j = i + 1; j < rk; ++j) s = __dadd_rn(s, -__dmul_rn(M[j][i], w[j]));
      w[i] = __ddiv_rn(s, M[i][i]);
    }
    for (int i = 0; i < r; ++i) a.z[i] = 0.0;
    for (int i = 0; i < rk; ++i) a.z[perm[i]] = w[i];
    const int k = a.ctl->iters + 1;
    a.ctl->iters = k;
    if (a.rec) a.rec[(size_t)k * REC + 2] = (double)rk;
  }
}

// p_j = sum_c Y[j, c] z[c] (ascending c), x_j += p_j
__global__ void __launch_bounds__(RP_NT) k_rp_update(RpArgs a) {
  if (rp_done(a)) return;
  __shared__ double zs[RP_RMAX];
  if (threadIdx.x < a.r) zs[threadIdx.x] = a.z[threadIdx.x];
  __syncthreads();
  const int r = a.r;
  for (int64_t j = (int64_t)blockIdx.x * RP_NT + threadIdx.x; j < a.n; j += (int64_t)gridDim.x * RP_NT) {
    const double* y = a.Y + j * r;
    double s = 0.0;
    for (int c = 0; c < r; ++c) s = __dadd_rn(s, __dmul_rn(y[c], zs[c]));
    a.p[j] = s;
    a.x[j] = __dadd_rn(a.x[j], s);
  }
}

}  // namespace plss
