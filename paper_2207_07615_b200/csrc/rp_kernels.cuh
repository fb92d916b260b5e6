// rp_kernels.cuh -- sm_100a device code of randomized projection ("Rand. Proj.", the paper's
// comparison method): eq:pkLong with W = I and a fresh
// random S_k in R^{m x r} every iteration (L171-176; Experiment I L985-991: standard normal, r = 10;
// Experiment III L1164-1170: sparse normal; Fig. 2: r = 10/20/40):
//
//   p_k = Y_k (Y_k^T Y_k)^+ S_k^T r_{k-1},  Y_k = A^T S_k,   x_k = x_{k-1} + p_k,  r_k = r_{k-1} - A p_k
//
// One iteration = five kernels here + K1 of the PLSS path (r <- r - A p, rho, stop test):
//   k_rp_gen    S_k (binary32, row-major m x ld, rows padded with zeros to ld = 8 ceil(r/8) floats
//               = whole 32-byte sectors) from the counter-based generator of DESIGN.md reading R17,
//               fused with the per-CTA partials of v = S_k^T r_{k-1} (fp64)
//   k_rp_spmm   Y_k = A^T S_k as a gather over the CSC copy: a group of G lanes per column loads G
//               (row, value) entries at once (coalesced), broadcasts them by shuffles and keeps 8
//               row gathers of S in flight per lane; lane c sums column c of Y sequentially in
//               ascending row order in fp64 (bitwise the oracle's per-column sequential sums)
//   k_rp_gram   per-CTA partials of the upper triangle of Y_k^T Y_k (fixed order)
//   k_rp_solve  one CTA: sums the partials in CTA order, pivoted Cholesky of the r x r Gram
//               matrix truncated at its numerical rank, z = M^+-equivalent solve (reading R18),
//               iteration counter
//   k_rp_update p = Y z, x <- x + p
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace plss {

constexpr int RP_RMAX = 64;        // largest sketch size r
constexpr int RP_NT = 256;
constexpr int RP_TILE = 4096;      // doubles of Y per shared-memory tile of the Gram kernel (32 KB)
constexpr int RP_PPT = (RP_RMAX * (RP_RMAX + 1) / 2 + RP_NT - 1) / RP_NT;   // Gram pairs per thread

// ---- counter-based sketch generator (reading R17; the oracle implements the same definition) ----
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
// ln(s), binary32 s in (0, 1), every op binary32 and correctly rounded (no contraction):
// frexp, m in [sqrt(1/2), sqrt(2)), f = (m-1)/(m+1), ln m = 2 f (1 + f^2/3 + ... + f^10/11) by
// Horner, ln s = e ln2 + ln m: bitwise the oracle's ln_unit32.
__device__ __forceinline__ float rp_ln32(float s) {
  int e;
  float mt = frexpf(s, &e);
  if (mt < __uint_as_float(0x3F3504F3u)) { mt = __fmul_rn(mt, 2.0f); e -= 1; }   // RN32(sqrt(1/2))
  const float f = __fdiv_rn(__fadd_rn(mt, -1.0f), __fadd_rn(mt, 1.0f));
  const float f2 = __fmul_rn(f, f);
  float t = 1.0f / 11.0f;
  t = __fadd_rn(__fmul_rn(t, f2), 1.0f / 9.0f);
  t = __fadd_rn(__fmul_rn(t, f2), 1.0f / 7.0f);
  t = __fadd_rn(__fmul_rn(t, f2), 1.0f / 5.0f);
  t = __fadd_rn(__fmul_rn(t, f2), 1.0f / 3.0f);
  t = __fadd_rn(__fmul_rn(t, f2), 1.0f);
  return __fadd_rn(__fmul_rn((float)e, __uint_as_float(0x3F317218u)), __fmul_rn(__fmul_rn(2.0f, f), t));
}
// (sin, cos)(2 pi u2), binary32, u2 in [0, 1) with 24-bit granularity: exact octant reduction,
// Taylor polynomials on [0, pi/4] by Horner (no contraction), octant symmetries; bitwise the
// oracle's sincos_2pi32.
__device__ __forceinline__ void rp_sincos_2pi32(float u2, float& sin_t, float& cos_t) {
  const float x = __fmul_rn(u2, 8.0f);
  const int o = (int)x;                                   // floor (x >= 0)
  float f = __fadd_rn(x, -(float)o);
  if (o & 1) f = __fadd_rn(1.0f, -f);
  const float phi = __fmul_rn(f, __uint_as_float(0x3F490FDBu));   // RN32(pi/4)
  const float p2 = __fmul_rn(phi, phi);
  float ts = 1.0f / 362880.0f;
  ts = __fadd_rn(__fmul_rn(ts, p2), -1.0f / 5040.0f);
  ts = __fadd_rn(__fmul_rn(ts, p2), 1.0f / 120.0f);
  ts = __fadd_rn(__fmul_rn(ts, p2), -1.0f / 6.0f);
  ts = __fadd_rn(__fmul_rn(ts, p2), 1.0f);
  const float sn = __fmul_rn(phi, ts);
  float cs = -1.0f / 3628800.0f;
  cs = __fadd_rn(__fmul_rn(cs, p2), 1.0f / 40320.0f);
  cs = __fadd_rn(__fmul_rn(cs, p2), -1.0f / 720.0f);
  cs = __fadd_rn(__fmul_rn(cs, p2), 1.0f / 24.0f);
  cs = __fadd_rn(__fmul_rn(cs, p2), -0.5f);
  cs = __fadd_rn(__fmul_rn(cs, p2), 1.0f);
  // octant symmetries without divergent branches (lanes hold random octants): swap sin / cos for
  // o in {1,2,5,6}, negate sin for o >= 4 and cos for o in {2,3,4,5} -- exact, so bitwise the
  // oracle's table (0: (s, c), 1: (c, s), 2: (c, -s), 3: (s, -c), 4: (-s, -c), 5: (-c, -s),
  // 6: (-c, s), 7: (-s, c))
  const bool swp = ((o + 1) >> 1) & 1;
  const float a = swp ? cs : sn, b = swp ? sn : cs;
  sin_t = o >= 4 ? -a : a;
  cos_t = (((o + 2) >> 2) & 1) ? -b : b;
}
// the binary32 normal pair (S[i, 2q], S[i, 2q+1]) of pair counter `base` = ((k 2^32 + i) h + q):
// Box-Muller from one 64-bit word (no rejection, so warps never diverge)
__device__ __forceinline__ void rp_pair(uint64_t key, uint64_t base, double density, float& z0, float& z1) {
  const uint64_t c = base * 256ull;
  const uint64_t w = rp_word(key, c);
  const float u1 = __fadd_rn(1.0f, -__fmul_rn((float)(uint32_t)(w >> 40), 0x1p-24f));
  const float u2 = __fmul_rn((float)(uint32_t)((w >> 16) & 0xFFFFFFull), 0x1p-24f);
  const float rad = __fsqrt_rn(__fmul_rn(-2.0f, rp_ln32(u1)));
  float sn, cs;
  rp_sincos_2pi32(u2, sn, cs);
  z0 = __fmul_rn(rad, cs);
  z1 = __fmul_rn(rad, sn);
  if (density < 1.0) {
    if (!(rp_unit(rp_word(key, c + 2ull)) < density)) z0 = 0.0f;
    if (!(rp_unit(rp_word(key, c + 3ull)) < density)) z1 = 0.0f;
  }
}

// Control shared with the PLSS path: the ctx's Ctl (iters, done, stop test via K1's tail_rho).
struct RpArgs {
  int64_t m, n;
  int32_t r, h;              // sketch size, pairs per row = ceil(r/2)
  int32_t ld;                // row stride of S in floats (even, >= r; 8 ceil(r/8) inside solves)
  uint64_t key;              // mix64(seed)
  double density;            // 1: dense normal S; < 1: each entry kept with this probability
  int64_t k_fixed;           // > 0: generate S_{k_fixed} (test entry point, no ctl)
  float* S;                  // m x ld row-major, binary32, columns >= r zero
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
  unsigned* colctr;          // k_rp_spmm's column-chunk counter (k_rp_gen of the step zeroes it)
  uint64_t pol_stream;       // L2 evict-first policy for the index / value streams
  Ctl* ctl;
  double* rec;
};

__device__ __forceinline__ bool rp_done(const RpArgs& a) { return a.ctl != nullptr && a.ctl->done; }

// S_k and v partials. CTA b owns rows [b*per, (b+1)*per); thread t -> pair q = t % h of rows
// lr = t / h, lr + rpp, ... (rpp = 256 / h rows per pass): consecutive threads write consecutive
// 8-byte pairs; the thread of the last pair also zeroes the row's padding [2h, ld), so whole
// padded rows are written. v partial of column c: sum over the CTA's threads of that column in
// lr order.
__global__ void __launch_bounds__(RP_NT) k_rp_gen(RpArgs a) {
  if (rp_done(a)) return;
  if (a.colctr && blockIdx.x == 0 && threadIdx.x == 0) *a.colctr = 0u;
  __shared__ double red[2][RP_NT];
  const int h = a.h, r = a.r, ld = a.ld;
  const int rpp = RP_NT / h;
  const int t = threadIdx.x, lr = t / h, q = t % h;
  const uint64_t k = a.k_fixed > 0 ? (uint64_t)a.k_fixed : (uint64_t)(a.ctl->iters + 1);
  const int64_t per = (a.m + gridDim.x - 1) / gridDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * per, i1 = min(a.m, i0 + per);
  const int c0 = 2 * q;
  const bool tail = q == h - 1;
  double acc0 = 0.0, acc1 = 0.0;
  if (lr < rpp) {
    for (int64_t i = i0 + lr; i < i1; i += rpp) {
      float z0, z1;
      rp_pair(a.key, ((k << 32) + (uint64_t)i) * (uint64_t)h + (uint64_t)q, a.density, z0, z1);
      if (c0 + 1 >= r) z1 = 0.0f;
      float* row = a.S + i * ld;
      *reinterpret_cast<float2*>(row + c0) = make_float2(z0, z1);
      if (tail)
        for (int c = 2 * h; c < ld; c += 2) *reinterpret_cast<float2*>(row + c) = make_float2(0.0f, 0.0f);
      if (a.res) {
        const double ri = a.res[i];
        acc0 = __dadd_rn(acc0, __dmul_rn((double)z0, ri));
        acc1 = __dadd_rn(acc1, __dmul_rn((double)z1, ri));
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

#ifndef PLSS_RP_PF
#define PLSS_RP_PF 64             // L2 prefetch-size qualifier on the S row gathers: with .L2::64B a
                                  // random row miss costs ~90 B of DRAM instead of ~160 B (uniform-
                                  // only probe: 79 vs 125 GB per A^T S), DESIGN.md section 13
#endif
__device__ __forceinline__ float rp_ld_s(const float* p) {
#if PLSS_RP_PF == 64
  float v;
  asm volatile("ld.global.nc.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
#elif PLSS_RP_PF == 128
  float v;
  asm volatile("ld.global.nc.L2::128B.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}
__device__ __forceinline__ int ld_stream_i32(const int32_t* p, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_stream_f64(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
template <int G, int CPL>
__global__ void __launch_bounds__(RP_NT) k_rp_spmm(RpArgs a) {
  if (rp_done(a)) return;
  constexpr int U = 8;                              // gathers in flight per lane (16: slower, more
                                                    // registers, fewer warps)
  constexpr int CPW = 32 / G;                       // columns per warp
  const int r = a.r, ld = a.ld;
  const int lane = threadIdx.x & 31;
  const int sub = lane / G, g = lane % G;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (sub * G));
  const uint64_t pol = a.pol_stream;
  // Columns are taken CPW at a time from a global counter: every warp works at the same moving
  // frontier, so the S rows of the band part of neighbouring columns are reused from L2 (a static
  // grid-stride split lets warps drift apart and loses that reuse).
  for (;;) {
    unsigned chunk = 0;
    if (lane == 0) chunk = atomicAdd(a.colctr, 1u);
    chunk = __shfl_sync(0xffffffffu, chunk, 0);
    const int64_t jb = (int64_t)chunk * CPW;
    if (jb >= a.n) break;
    const int64_t j = jb + sub;
    int b = 0, e = 0;
    if (j < a.n) { b = __ldg(a.col_ptr + j); e = __ldg(a.col_ptr + j + 1); }
    double acc[CPL];
#pragma unroll
    for (int u = 0; u < CPL; ++u) acc[u] = 0.0;
    int ci = 0;
    double cv = 0.0;
    if (b + g < e) { ci = ld_stream_i32(a.row_idx + b + g, pol); cv = ld_stream_f64(a.val_t + b + g, pol); }
    for (int t0 = b; t0 < e; t0 += G) {             // uniform within the group
      int ni = 0;
      double nv = 0.0;
      if (t0 + G + g < e) { ni = ld_stream_i32(a.row_idx + t0 + G + g, pol); nv = ld_stream_f64(a.val_t + t0 + G + g, pol); }
      const int cnt = min(G, e - t0);
#pragma unroll
      for (int u0 = 0; u0 < G; u0 += U) {
        if (u0 >= cnt) break;
        float sv[U][CPL];
        double vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int iu = __shfl_sync(gmask, ci, u0 + u, G);
          vv[u] = __shfl_sync(gmask, cv, u0 + u, G);
#pragma unroll
          for (int w = 0; w < CPL; ++w) {
            const int c = g + w * G;
            sv[u][w] = (u0 + u < cnt && c < r) ? rp_ld_s(a.S + (int64_t)iu * ld + c) : 0.0f;
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (u0 + u < cnt) {
#pragma unroll
            for (int w = 0; w < CPL; ++w) acc[w] = __dadd_rn(acc[w], __dmul_rn(vv[u], (double)sv[u][w]));
          }
        }
      }
      ci = ni;
      cv = nv;
    }
    if (j < a.n) {
#pragma unroll
      for (int w = 0; w < CPL; ++w) {
        const int c = g + w * G;
        if (c < r) __stcs(a.Y + j * r + c, acc[w]);
      }
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
// null(M) = null(Y), so Y z equals Y M^+ v (reading R18).
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
