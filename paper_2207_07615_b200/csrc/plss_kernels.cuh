// plss_kernels.cuh -- sm_100a device code of the PLSS hot path (arXiv 2207.07615, Algorithm 1,
// PAPER.md L773-816, WI = I). fp64 CUDA-core kernels: the path is two bandwidth-bound SpMVs
// plus streaming vector ops (~0.17 flop/B), so no tensor cores are involved.
//
//   K1  k_spmv<ROLE_K1>  r <- r - A p over CSR (eq:recRes L663-666, Alg.1) fused with the
//                        rho = r^T r reduction (L804) and, in its last CTA, the stop test
//                        sqrt(rho)/||b|| <= tol (L828-831 / L977) and the history record.
//   K2  k_spmv<ROLE_K2 / ROLE_K2DOTS> y = A^T r as a GATHER over the CSC copy (L802; no atomics, so every
//                        sum has a fixed order) fused with phi = y^T y (L806) and
//                        psi = y^T p_{k-1} (L671-672), and in its last CTA the scalar tail
//                        tau, beta, gamma (L807-809).
//   K3  k_pxupdate       p <- beta p + gamma y (Thm 4.1 eq:pkShort), theta = p^T p, x <- x + p
//                        (L811-813).
//
// Every SpMV output element is a SEQUENTIAL sum in ascending index order computed with
// __dmul_rn/__dadd_rn (no FMA contraction): products and sums are bitwise those of the plain
// oracle. Dot products use fixed-shape trees: deterministic run to run, a few ulps from the
// oracle's sequential sums.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace plss {

constexpr int NT = 256;            // threads per CTA of the SpMV / vector kernels
constexpr int TILE = 2048;         // nnz per SpMV tile (owner-computes rows starting in it)
constexpr int CAP = TILE + 512;    // staged products per tile (spill of the last row)
constexpr int UNR = CAP / NT;      // staged loads per thread (10)
constexpr int LONGROW = 32;        // rows longer than this are summed by the whole warp
constexpr int REC = 8;             // doubles per iteration record
constexpr unsigned FULL = 0xffffffffu;

enum { OUT_CONVERGED = 0, OUT_MAXIT = 1, OUT_Y_VANISHED = 2, OUT_STAGNATION = 3,
       OUT_RUNNING = -1 };

// Device-resident control block: the whole loop state lives on the device so the host never
// synchronizes per iteration (CUDA graphs run chunks of iterations; kernels no-op once done).
struct Ctl {
  double nbd;       // denominator of the stop test: ||b|| (relative) or 1
  double tol;
  double freeze_h;  // freeze threshold on hist (64 eps)
  double rho, phi, psi, theta, beta, gamma;
  double nb2;       // ||b||^2 (local on a rank before the all-reduce)
  int32_t iters, maxit, done, frozen, stopped, outcome, freeze, tol_mode;
};

enum Role { ROLE_PLAIN = 0, ROLE_K1 = 1, ROLE_K2 = 2, ROLE_K2DOTS = 3 };

// One SpMV launch over a "segment": a CSR (K1) or CSC (K2) slab, tiled by nnz.
struct SpmvSeg {
  const int32_t* ptr;        // nrows+1 absolute positions into idx / val
  const int32_t* idx;        // gathered-vector index of each entry (column for K1, row for K2)
  const double* val;
  const int32_t* tile_first; // ntiles+1: tile t owns rows whose first entry lies in
                             // [e0 + t*TILE, e0 + (t+1)*TILE)
  long long e0;
  int32_t nrows, ntiles;
  const double* g;           // gathered vector (p for K1, the slab of r for K2)
  double* out;               // r (K1, read-modify-write) / y (K2) / result (plain)
  const double* pv;          // p, for psi (K2DOTS)
  double* partial;           // this launch's per-CTA partial pairs
  double* part_base;         // all partial pairs reduced by the finalizing CTA
  int32_t nparts;            // number of pairs at part_base
  int32_t accumulate;        // K2: continue the sum from out[i] (slab s > 0)
  int32_t finalize;          // this launch elects a last CTA that runs the tail
  int32_t dist;              // distributed: K1 tail publishes the local rho instead
  unsigned* counter;
  Ctl* ctl;
  double* rec;
  double* rho_out;           // dist: where the local rho goes (all-reduce buffer [n])
};

// ---------------------------------------------------------------------------------------------
// memory helpers
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// Streaming (read-once) loads of the matrix arrays: no L1 allocation, L2 evict-first, so the
// gathered vector keeps its L2 residency.
__device__ __forceinline__ double ld_stream(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t* p, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
               : "=r"(v) : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);  // butterfly: same in all lanes
  return v;
}

// Fixed-shape block reduction of two values; result valid in thread 0.
__device__ __forceinline__ void block_sum2(double& a, double& b, double (*sm)[NT / 32]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  if (lane == 0) { sm[0][warp] = a; sm[1][warp] = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) { s0 += sm[0][w]; s1 += sm[1][w]; }
    a = s0; b = s1;
  }
  __syncthreads();
}

// Last-CTA election. Every CTA publishes its partial pair; the CTA that arrives last
// (atomic ticket) sums ALL pairs in index order -- the ticket decides only who sums, never the
// order, so the result is deterministic. Returns true in every thread of the last CTA, with
// (a, b) = totals in thread 0.
__device__ __forceinline__ bool publish_and_elect(double& a, double& b, double* partial,
                                                  const double* part_base, int nparts,
                                                  unsigned* counter, double (*sm)[NT / 32]) {
  __shared__ int s_last;
  block_sum2(a, b, sm);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = a;
    partial[2 * blockIdx.x + 1] = b;
    __threadfence();
    unsigned prev = atomicAdd(counter, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  double s0 = 0.0, s1 = 0.0;
  for (int q = threadIdx.x; q < nparts; q += NT) {
    s0 += __ldcg(part_base + 2 * q);
    s1 += __ldcg(part_base + 2 * q + 1);
  }
  block_sum2(s0, s1, sm);
  if (threadIdx.x == 0) { a = s0; b = s1; *counter = 0u; }
  return true;
}

// ---------------------------------------------------------------------------------------------
// scalar tails (one thread). Exactly Algorithm 1's operation order, correctly rounded
// intrinsics, no contraction: bitwise equal to the oracle for equal inputs.
// ---------------------------------------------------------------------------------------------
__device__ void tail_rho(Ctl* c, double* rec, double rho) {
  const int k = c->iters;
  const double h = __ddiv_rn(__dsqrt_rn(rho), c->nbd);        // sqrt(rho_k)/||b||
  c->rho = rho;
  rec[(size_t)k * REC + 0] = h;
  rec[(size_t)k * REC + 1] = rho;
  if (rho == 0.0 || h <= c->tol) {                             // stop test (L828-831, L977)
    if (!c->freeze) { c->done = 1; c->outcome = OUT_CONVERGED; return; }
    if (!c->stopped) { c->outcome = OUT_CONVERGED; c->stopped = 1; }
    c->frozen = 1;
  } else if (c->freeze && h <= c->freeze_h) {
    c->frozen = 1;
  }
}

__device__ void guard(Ctl* c, int outcome) {
  if (!c->freeze) { c->done = 1; c->outcome = outcome; return; }
  if (!c->stopped) { c->outcome = outcome; c->stopped = 1; }
  c->frozen = 1;
}

__device__ void tail_y(Ctl* c, double* rec, double phi, double psi) {
  const int k = c->iters;
  double* rk = rec + (size_t)k * REC;
  if (k == 0) {                                                // initialization (L786-797)
    if (phi <= 1e-300) { guard(c, OUT_Y_VANISHED); if (c->done) return; }
    const double g0 = c->frozen ? 0.0 : __ddiv_rn(c->rho, phi); // p1 = (rho/phi) y
    c->phi = phi; c->beta = 0.0; c->gamma = g0;
    rk[2] = phi; rk[7] = g0;
    return;
  }
  double tau = 0.0, beta = 0.0, gamma = 0.0;
  if (!c->frozen) {
    tau = __ddiv_rn(__dsqrt_rn(__dmul_rn(c->theta, phi)), c->rho);          // L807
    if (phi <= 1e-300) {
      guard(c, OUT_Y_VANISHED);
    } else if (__dadd_rn(tau, -1.0) <= 1e-14) {
      guard(c, OUT_STAGNATION);
    } else {
      beta = __ddiv_rn(1.0, __dmul_rn(__dadd_rn(tau, -1.0), __dadd_rn(tau, 1.0)));  // L807-808
      gamma = __dmul_rn(__ddiv_rn(c->theta, c->rho), beta);                        // L809
    }
    if (c->done) return;
  }
  c->phi = phi; c->psi = psi; c->beta = beta; c->gamma = gamma;
  rk[2] = phi; rk[3] = psi; rk[5] = tau; rk[6] = beta; rk[7] = gamma;
}

// ---------------------------------------------------------------------------------------------
// K1 / K2 / plain SpMV: persistent CTAs over nnz tiles, products staged in shared memory,
// rows owned by the tile holding their first entry, sequential per-row sums.
// ---------------------------------------------------------------------------------------------
template <int ROLE>
__global__ void __launch_bounds__(NT) k_spmv(SpmvSeg a) {
  __shared__ double prod[CAP];
  __shared__ double sm[2][NT / 32];
  if (a.ctl != nullptr && a.ctl->done) return;
  const uint64_t pol = policy_evict_first();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double acc0 = 0.0, acc1 = 0.0;

  for (int t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
    const int r0 = a.tile_first[t], r1 = a.tile_first[t + 1];
    if (r0 >= r1) continue;                                    // uniform in the CTA
    const long long s0 = a.ptr[r0];
    const long long s1 = a.ptr[r1];
    const int cnt = (int)min(s1 - s0, (long long)CAP);
    const long long send = s0 + cnt;
    // stage: coalesced streaming loads of the tile's values and indices, then the gathers
    double v[UNR];
    int32_t c[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int k = tid + u * NT;
      if (k < cnt) { v[u] = ld_stream(a.val + s0 + k, pol); c[u] = ld_stream(a.idx + s0 + k, pol); }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int k = tid + u * NT;
      if (k < cnt) prod[k] = __dmul_rn(v[u], __ldg(a.g + c[u]));
    }
    __syncthreads();
    for (int base = r0 + warp * 32; base < r1; base += NT) {
      const int i = base + lane;
      const bool valid = i < r1;
      long long b = 0, e = 0;
      if (valid) { b = a.ptr[i]; e = a.ptr[i + 1]; }
      const bool lng = valid && (e - b) > LONGROW;
      double s = 0.0;
      if (ROLE >= ROLE_K2 && valid && a.accumulate) s = a.out[i];
      if (valid && !lng) {
        for (long long k = b; k < e; ++k) {
          const double pr = (k < send) ? prod[k - s0]
                                       : __dmul_rn(ld_stream(a.val + k, pol), __ldg(a.g + ld_stream(a.idx + k, pol)));
          s = __dadd_rn(s, pr);
        }
      }
      unsigned mask = __ballot_sync(FULL, lng);
      while (mask) {                                            // warp-cooperative long rows
        const int l = __ffs(mask) - 1;
        mask &= mask - 1;
        const long long lb = __shfl_sync(FULL, b, l), le = __shfl_sync(FULL, e, l);
        double ps = 0.0;
        for (long long k = lb + lane; k < le; k += 32) {
          const double pr = (k < send) ? prod[k - s0]
                                       : __dmul_rn(ld_stream(a.val + k, pol), __ldg(a.g + ld_stream(a.idx + k, pol)));
          ps = __dadd_rn(ps, pr);
        }
        ps = warp_sum(ps);
        if (lane == l) s = __dadd_rn(s, ps);
      }
      if (valid) {
        if (ROLE == ROLE_PLAIN) {
          a.out[i] = s;
        } else if (ROLE == ROLE_K1) {
          const double rn = __dsub_rn(a.out[i], s);            // r_i <- r_i - (A p)_i
          a.out[i] = rn;
          acc0 = fma(rn, rn, acc0);
        } else {
          a.out[i] = s;                                         // y_j
          if (ROLE == ROLE_K2DOTS) { acc0 = fma(s, s, acc0); acc1 = fma(s, a.pv[i], acc1); }
        }
      }
    }
    __syncthreads();
  }
  if (ROLE == ROLE_PLAIN || ROLE == ROLE_K2) return;           // nothing to reduce
  if (!a.finalize) {                                            // slab s < S-1: publish only
    block_sum2(acc0, acc1, sm);
    if (tid == 0) { a.partial[2 * blockIdx.x] = acc0; a.partial[2 * blockIdx.x + 1] = acc1; }
    return;
  }
  if (!publish_and_elect(acc0, acc1, a.partial, a.part_base, a.nparts, a.counter, sm)) return;
  if (tid != 0) return;
  if (ROLE == ROLE_K1) {
    if (a.dist) *a.rho_out = acc0;                              // local rho -> all-reduce buffer
    else tail_rho(a.ctl, a.rec, acc0);
  } else if (ROLE == ROLE_K2DOTS) {
    tail_y(a.ctl, a.rec, acc0, acc1);
  }
}

// ---------------------------------------------------------------------------------------------
// K3: p <- beta p + gamma y; theta = p^T p; x <- x + p  (L811-813); init: p = gamma y (L795)
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) k_pxupdate(double* __restrict__ p, const double* __restrict__ y,
                                                 double* __restrict__ x, long long n, Ctl* c,
                                                 double* rec, double* partial, unsigned* counter) {
  __shared__ double sm[2][NT / 32];
  if (c->done) return;
  const int k = c->iters;
  const bool init = (k == 0);
  const double beta = c->beta, gamma = c->gamma;
  double acc = 0.0, dummy = 0.0;
  const long long n2 = n >> 1;
  const long long stride = (long long)gridDim.x * NT;
  double2* p2 = reinterpret_cast<double2*>(p);
  double2* x2 = reinterpret_cast<double2*>(x);
  const double2* y2 = reinterpret_cast<const double2*>(y);
  for (long long i = (long long)blockIdx.x * NT + threadIdx.x; i < n2; i += stride) {
    const double2 yy = __ldcs(y2 + i);
    double2 pp;
    if (init) {
      pp.x = __dmul_rn(gamma, yy.x);
      pp.y = __dmul_rn(gamma, yy.y);
    } else {
      const double2 po = p2[i];
      pp.x = __dadd_rn(__dmul_rn(beta, po.x), __dmul_rn(gamma, yy.x));
      pp.y = __dadd_rn(__dmul_rn(beta, po.y), __dmul_rn(gamma, yy.y));
    }
    p2[i] = pp;
    double2 xx = __ldcs(x2 + i);
    xx.x = __dadd_rn(xx.x, pp.x);
    xx.y = __dadd_rn(xx.y, pp.y);
    __stcs(x2 + i, xx);
    acc = fma(pp.x, pp.x, acc);
    acc = fma(pp.y, pp.y, acc);
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const long long i = n - 1;
    const double pp = init ? __dmul_rn(gamma, y[i]) : __dadd_rn(__dmul_rn(beta, p[i]), __dmul_rn(gamma, y[i]));
    p[i] = pp;
    x[i] = __dadd_rn(x[i], pp);
    acc = fma(pp, pp, acc);
  }
  if (!publish_and_elect(acc, dummy, partial, partial, gridDim.x, counter, sm)) return;
  if (threadIdx.x != 0) return;
  c->theta = acc;                                               // theta = p^T p (L812)
  rec[(size_t)k * REC + 4] = acc;
  c->iters = k + 1;
  if (k + 1 >= c->maxit) {
    c->done = 1;
    if (!c->stopped) c->outcome = OUT_MAXIT;
  }
}

// ---------------------------------------------------------------------------------------------
// distributed: phi, psi over the replicated (all-reduced) y, then both tails (K2b)
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) k_dots_tail(const double* __restrict__ y, const double* __restrict__ p,
                                                  long long n, const double* rho_g, Ctl* c,
                                                  double* rec, double* partial, unsigned* counter) {
  __shared__ double sm[2][NT / 32];
  if (c->done) return;
  double a0 = 0.0, a1 = 0.0;
  for (long long i = (long long)blockIdx.x * NT + threadIdx.x; i < n; i += (long long)gridDim.x * NT) {
    const double yy = y[i];
    a0 = fma(yy, yy, a0);
    a1 = fma(yy, p[i], a1);
  }
  if (!publish_and_elect(a0, a1, partial, partial, gridDim.x, counter, sm)) return;
  if (threadIdx.x != 0) return;
  tail_rho(c, rec, *rho_g);
  if (c->done) return;
  tail_y(c, rec, a0, a1);
}

// ||b||^2 (or the local share of it) into ctl->nb2; non-dist also sets nbd.
__global__ void __launch_bounds__(NT) k_norm_b(const double* __restrict__ r, long long m, Ctl* c,
                                               double* partial, unsigned* counter, int set_nbd,
                                               double* out) {
  __shared__ double sm[2][NT / 32];
  double a0 = 0.0, a1 = 0.0;
  for (long long i = (long long)blockIdx.x * NT + threadIdx.x; i < m; i += (long long)gridDim.x * NT)
    a0 = fma(r[i], r[i], a0);
  if (!publish_and_elect(a0, a1, partial, partial, gridDim.x, counter, sm)) return;
  if (threadIdx.x != 0) return;
  c->nb2 = a0;
  if (out) *out = a0;
  if (set_nbd) {
    const double nb = __dsqrt_rn(a0);
    c->nbd = (c->tol_mode == 0 && nb > 0.0) ? nb : 1.0;
  }
}

__global__ void k_set_nbd(Ctl* c, const double* nb2) {
  const double nb = __dsqrt_rn(*nb2);
  c->nb2 = *nb2;
  c->nbd = (c->tol_mode == 0 && nb > 0.0) ? nb : 1.0;
}

// ---------------------------------------------------------------------------------------------
// setup kernels (once per ctx)
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ int lower_bound_pos(const int32_t* ptr, int nrows, long long key) {
  int lo = 0, hi = nrows;
  while (lo < hi) {
    const int mid = lo + ((hi - lo) >> 1);
    if ((long long)ptr[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_tile_map(const int32_t* ptr, int nrows, long long e0, int ntiles, int32_t* tf) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > ntiles) return;
  if (t == 0) tf[0] = 0;
  else if (t == ntiles) tf[t] = nrows;
  else tf[t] = lower_bound_pos(ptr, nrows, e0 + (long long)t * TILE);
}

// structural validation of one compressed layout (CSR or CSC); bit flags into *err
__global__ void k_validate(const int32_t* ptr, const int32_t* idx, const double* val, long long nrows,
                           long long ncols, long long nnz, int* err) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0 && (ptr[0] != 0 || (long long)ptr[nrows] != nnz)) atomicOr(err, 1);
  if (i >= nrows) return;
  const long long b = ptr[i], e = ptr[i + 1];
  if (e < b || b < 0 || e > nnz) { atomicOr(err, 2); return; }
  for (long long k = b; k < e; ++k) {
    const int32_t j = idx[k];
    if (j < 0 || j >= ncols) { atomicOr(err, 4); return; }
    if (k > b && idx[k - 1] >= j) { atomicOr(err, 8); return; }
    if (!isfinite(val[k])) { atomicOr(err, 16); return; }
  }
}

// every CSC entry (j, i, v) must be the CSR entry (i, j, v)  => CSC == CSR^T (equal nnz)
__global__ void k_validate_pair(const int32_t* row_ptr, const int32_t* col_idx, const double* val,
                                const int32_t* col_ptr, const int32_t* row_idx, const double* val_t,
                                long long n, int* err) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  for (long long k = col_ptr[j]; k < col_ptr[j + 1]; ++k) {
    const int32_t i = row_idx[k];
    long long lo = row_ptr[i], hi = row_ptr[i + 1];
    while (lo < hi) {
      const long long mid = lo + ((hi - lo) >> 1);
      if (col_idx[mid] < j) lo = mid + 1; else hi = mid;
    }
    if (lo >= row_ptr[i + 1] || col_idx[lo] != j ||
        __double_as_longlong(val[lo]) != __double_as_longlong(val_t[k])) {
      atomicOr(err, 32);
      return;
    }
  }
}

// slab-major CSC: count entries of column j whose row lies in [R0, R1)
__device__ __forceinline__ long long col_lb(const int32_t* row_idx, long long b, long long e, long long key) {
  while (b < e) {
    const long long mid = b + ((e - b) >> 1);
    if ((long long)row_idx[mid] < key) b = mid + 1; else e = mid;
  }
  return b;
}

__global__ void k_slab_count(const int32_t* col_ptr, const int32_t* row_idx, long long n, long long R0,
                             long long R1, int32_t* cnt) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j > n) return;
  if (j == n) { cnt[n] = 0; return; }
  const long long b = col_ptr[j], e = col_ptr[j + 1];
  cnt[j] = (int32_t)(col_lb(row_idx, b, e, R1) - col_lb(row_idx, b, e, R0));
}

__global__ void k_slab_copy(const int32_t* col_ptr, const int32_t* row_idx, const double* val_t,
                            long long n, long long R0, long long R1, long long E0, int32_t* sptr,
                            int32_t* sidx, double* sval) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j > n) return;
  const long long dst = (long long)sptr[j] + E0;
  sptr[j] = (int32_t)dst;                                      // make the scan absolute
  if (j == n) return;
  const long long b = col_ptr[j], e = col_ptr[j + 1];
  const long long s = col_lb(row_idx, b, e, R0), t = col_lb(row_idx, b, e, R1);
  for (long long k = s; k < t; ++k) {
    sidx[dst + (k - s)] = (int32_t)(row_idx[k] - R0);
    sval[dst + (k - s)] = val_t[k];
  }
}

}  // namespace plss
