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
// Every SpMV output element of a row (column) with <= LONGROW entries is a SEQUENTIAL sum in
// ascending index order computed with __dmul_rn/__dadd_rn (no FMA contraction): bitwise the
// oracle's. Longer rows are summed by a whole warp (lane-strided partials + butterfly):
// deterministic, within a few ulps of the sequential sum. Dot products use fixed-shape trees: deterministic run to run, a few ulps from the
// oracle's sequential sums.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <cub/block/block_radix_sort.cuh>

namespace plss {

#ifndef PLSS_TILE
#define PLSS_TILE 1024
#endif
#ifndef PLSS_NST
#define PLSS_NST 2
#endif
#ifndef PLSS_MINB
#define PLSS_MINB 4
#endif
constexpr int NT = 256;                 // threads per CTA of the vector kernels
constexpr int NCW = 8;                  // warps per CSR-tile SpMV CTA
constexpr int NTS = NT;                 // CSR-tile CTA: 8 warps, thread 0 also issues the TMA copies
constexpr int TILE = PLSS_TILE;         // nnz window of a SpMV tile (rows whose first entry lies in it)
constexpr int SUBW = TILE / NCW;        // nnz sub-window of one consumer warp
constexpr int RCAP = TILE / 4;          // at most this many rows per tile
#ifndef PLSS_ABLATE
#define PLSS_ABLATE 0       // timing experiments only: 1 = no gathers, 2 = no row phase
#endif
#ifndef PLSS_SLACK
#define PLSS_SLACK (PLSS_TILE / 4)
#endif
constexpr int CAP = TILE + PLSS_SLACK;  // staged entries per tile (the last row may spill past TILE)
constexpr int WUNR = 4;                 // gathers in flight per lane per batch
constexpr int NST = PLSS_NST;           // TMA pipeline stages per CTA
constexpr int MINB = PLSS_MINB;         // CTAs per SM the SpMV kernel is compiled for
constexpr int LONGROW = 128;       // rows longer than this are summed by the whole warp (tree)
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
  int32_t weighted; // PLSS W: WI = diag(wi) (Algorithm 1 with B^T B)
  int32_t xlag;     // K3_XDEFER: x lacks the current p (x_k = x + p); plss_finish applies it
};

enum Role { ROLE_PLAIN = 0, ROLE_K1 = 1, ROLE_K2 = 2, ROLE_K2DOTS = 3 };

// One SpMV launch over a "segment": a CSR (K1) or CSC (K2) slab, tiled by nnz.
struct SpmvSeg {
  const int32_t* ptr;        // nrows+1 absolute positions into idx / val
  const int32_t* idx;        // gathered-vector index of each entry (column for K1, row for K2)
  const double* val;
  const int2* desc;          // ntiles+1 tile descriptors {first row, its first entry}; a tile
                             // is a maximal run of <= RCAP rows whose first entries share one
                             // TILE-wide window of positions (counted from e0)
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
  // SELL-32 format (fmt = 1): slice s holds rows perm[32s .. 32s+31] column-major, entry j of
  // its lane l at (sptr[s] + j) * 32 + l; padding entries have index -1
  int32_t fmt;               // 0: CSR tiles through TMA (k_spmv), 1: SELL-32 (k_sell),
                             // 2: SELL-32 + shared-memory window of g (k_sellw), 3: SELL-32 over
                             // per-SM slice ranges (k_sell<.., 1024>), 5: a thread per short row
                             // over the original arrays (k_scalar)
  int32_t nslices;
  const int32_t* sptr;       // nslices+1 slice starts in 32-entry steps
  const int32_t* perm;       // slot -> segment-local row (sigma-sorted), -1 for padding; or NULL
  // window (fmt = 2): blocks of NSB consecutive slices; block b gathers g[lo_b, lo_b + win) from a
  // ring of `ring` doubles in shared memory, every other entry from global memory
  int32_t win, ring, nblocks, glen, nsb;
  int32_t row0;              // first row of this segment in the matrix (ablation experiments only)
  int32_t sig;               // sigma window of this segment's sort: 0 = SIGMA, or SIGMA_WIDE (K2
                             // segments whose SIGMA windows leave too much padding, C4's columns)
  int32_t wrow0;             // first row of the segment's sigma window 0 (0; a column chunk of a K2
                             // segment, see plss.cu make_chunks, starts at a later window)
  // Globally length-sorted SELL (power-law rows, fmt 3 only): perm is a global row order; the nlong
  // rows longer than LONGROW are not in the slices but run in k_longrows, one CTA per row (row
  // lrows[k], entries of the segment's CSR-like arrays lidx / lval)
  int32_t gsort, nlong;
  const int32_t* lrows;
  const int32_t* lptr;
  // k_longrows (launch_spmv runs it after the segment's slices): per long row its dot terms
  // (2 doubles, reduced in row order by the last CTA) and that CTA's election counter
  double* lrowd;
  unsigned* lcounter;
  // k_longrows runs concurrently with the segment's slices (launch_spmv forks it onto a second
  // stream): the slices' CTAs and k_longrows' last CTA (elect_extra = 1 arrival) elect together the
  // CTA that finalizes; elect_total = the slices' grid + 1
  int32_t elect_extra, elect_total;
  int32_t psi3;              // K2's finalizing segment on one device: psi left to K3 (k2_final)
  int32_t scb;               // fmt 5: entries per thread in flight (k_scalar's SCBT: 2 or 3)
  long long long_entries, short_entries;   // setup: entries of the long rows / of the slices
  void* fork_stream;         // host handles (cudaStream_t, cudaEvent_t x 2) for that fork / join
  void* fork_ev;
  void* join_ev;
  const int32_t* lbeg;       // k_longrows: entry range [lbeg[2k], lbeg[2k+1]) of long row k (absolute
                             // positions; setup orders the long rows by length, longest first)
  
  const int32_t* lidx;
  const double* lval;
  // k_longchunks (the default for long rows): long row k split into chunks of LCH entries, chunk c
  // = {e0, e1, k, first chunk of row k} (rows longest first, a row's chunks consecutive); a warp
  // per chunk; lnch[k] chunks of row k; lrcnt[k] its finished chunks (the warp finishing the last
  // one sums the row's chunk partials lcpart[] in chunk order and resets it); NULL: k_longrows
  const int4* lchunk;
  const int32_t* lnch;
  unsigned* lrcnt;
  double* lcpart;
  int32_t nchunks;
  // row dot terms reduced in two fixed levels: groups of 32 rows (lgcnt[g]: finished rows of group
  // g; its last finisher sums lrowd over the group into lgd[g]), then the ngroup group sums
  unsigned* lgcnt;
  double* lgd;
  const int32_t* uw;         // nunits+1 prefix of stored entries per unit (CTA balance), or NULL
  // L2 cache policies (createpolicy values computed once at setup by k_policies). Passed as kernel
  // parameters they sit in uniform registers: a per-thread createpolicy result costs one R2UR
  // (XU pipe) per cache-hinted load, which saturated the XU pipe of K1 (profiles/r01_notes.md).
  uint64_t pol_first, pol_last;
  const double* wi;          // K2's last slab: the diagonal of WI (used when ctl->weighted)
  const int2* wlo;           // per block {lo_b, flags}: 1 = reload the whole window, 2 = no window
  const int32_t* cblk;       // grid+1 block bounds of the CTAs (balanced by stored entries)
  double* slpart;            // per-slice dot partials (fixed-order reduction, deterministic)
  unsigned long long* ctat;  // diagnostics (a -DPLSS_DBGCTA build with PLSS_DBG_CTA=1, plss_debug_cta_times): per CTA of fmt 3 its
                             // start / end %globaltimer, stored entries and units processed; or NULL
  int32_t stat;              // fmt 3 without perm / long rows: warps step through their CTA's slices
                             // statically and keep per-thread dot terms (no per-slice partials);
                             // 2: the same with 6 entries per lane in flight (slices of 6 k steps)
  // Globally sorted segments: the tail of slices of one step (rows of one entry: 64% of C4's rows)
  // and of no step (empty rows) runs in batches of S1B slices per warp (k_sell's second phase):
  // slices [s1beg, s1end) have one step each, slice t's at step s1step0 + t - s1beg; slices from
  // s1end on have none. s1on = 0: no such phase.
  int32_t s1on, s1beg, s1end, s1step0;
  // Globally sorted segments with long rows in chunks: 1 = k_sell runs the chunks itself (phase 0),
  // 0 = a concurrent k_longchunks launch
  int32_t lin;
};

// ---------------------------------------------------------------------------------------------
// memory helpers
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_stream(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ double ld_hint(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
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

// K2's last slab (phi, psi): y_j = s gives phi's term y_j WIy_j and psi's y_j p_j; returns what K3
// consumes, WIy_j = y_j / wi_j under PLSS W (WI \\ y applied element-wise, L805, L819-821), else y_j.
// psi3 (one device, WI = I): psi is summed by K3, which reads y and p_{k-1} coalesced anyway, so K2
// reads no p (C5's last slab: scattered per sigma window; C4's columns: 64 MB)
__device__ __forceinline__ double k2_final(const SpmvSeg& a, bool wtd, long long row, double s, double& d0,
                                           double& d1) {
  if (wtd) {
    const double wy = __ddiv_rn(s, a.wi[row]);
    d0 = s * wy;
    d1 = s * a.pv[row];
    return wy;
  }
  d0 = s * s;
  d1 = a.psi3 ? 0.0 : s * a.pv[row];
  return s;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);  // butterfly: same in all lanes
  return v;
}

// Fixed-shape block reduction of two values; result valid in thread 0.
constexpr int MAXW = 32;  // max warps per CTA of any kernel here

__device__ __forceinline__ void block_sum2(double& a, double& b, double (*sm)[MAXW]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  if (lane == 0) { sm[0][warp] = a; sm[1][warp] = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { s0 += sm[0][w]; s1 += sm[1][w]; }
    a = s0; b = s1;
  }
  __syncthreads();
}

// Streaming vector kernels (K3, the norms): at least 6 CTAs of NT threads per SM (<= 40 registers,
// no spills). Their finalizing sum (final_sum2's 8 loads in flight) otherwise raised k_pxupdate to
// 62 registers and 4 CTAs per SM (C4's K3 0.056 -> 0.065 ms); the dots kernels of the distributed
// steps would spill ~100 bytes under the bound and keep their own.
#ifndef PLSS_VEC_MINB
#define PLSS_VEC_MINB 6
#endif
constexpr int VEC_MINB = PLSS_VEC_MINB;

// The finalizing sum of all partial pairs, in one fixed shape whatever the CTA size (>= FIN_NT
// threads): thread t < FIN_NT sums pairs t, t + FIN_NT, ... sequentially, each warp butterflies,
// thread 0 adds the FIN_NT / 32 warp sums in order. A k_sell CTA (1024 threads) and a k_longchunks
// warp (fin_sum2_warp) reach bitwise the same totals, so it does not matter which one finalizes.
constexpr int FIN_NT = 256;
// s0 += base[2q], s1 += base[2q + 1] for q = q0, q0 + step, ... < n in that order (the plain
// sequential sum), with the loads issued 8 at a time: the serial tails of one warp (k_longchunks)
// otherwise wait for one L2 round trip per term. Out-of-range terms add +0.0, an exact identity
// here (a sum started at +0.0 never becomes -0.0 under round-to-nearest).
__device__ __forceinline__ void seq_add2(const double* base, int q0, int n, int step, double& s0, double& s1) {
  for (int q = q0; q < n; q += 8 * step) {
    double x0[8], x1[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int qq = q + u * step;
      x0[u] = qq < n ? __ldcg(base + 2 * qq) : 0.0;
      x1[u] = qq < n ? __ldcg(base + 2 * qq + 1) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) { s0 += x0[u]; s1 += x1[u]; }
  }
}
__device__ __forceinline__ void final_sum2(const double* part_base, int nparts, double& a, double& b,
                                           double (*sm)[MAXW]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int F = blockDim.x < FIN_NT ? blockDim.x : FIN_NT;
  double s0 = 0.0, s1 = 0.0;
  if (threadIdx.x < F) seq_add2(part_base, threadIdx.x, nparts, F, s0, s1);
  s0 = warp_sum(s0);
  s1 = warp_sum(s1);
  __syncthreads();                                   // sm may still be read by an earlier block_sum2
  if (lane == 0) { sm[0][warp] = s0; sm[1][warp] = s1; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t0 = 0.0, t1 = 0.0;
    for (int w = 0; w < F / 32; ++w) { t0 += sm[0][w]; t1 += sm[1][w]; }
    a = t0; b = t1;
  }
}
// the same shape computed by one warp (every lane returns the totals)
__device__ __forceinline__ void final_sum2_warp(const double* part_base, int nparts, double& a, double& b) {
  const int lane = threadIdx.x & 31;
  double t0 = 0.0, t1 = 0.0;
  for (int w = 0; w < FIN_NT / 32; ++w) {
    double s0 = 0.0, s1 = 0.0;
    seq_add2(part_base, w * 32 + lane, nparts, FIN_NT, s0, s1);
    t0 += warp_sum(s0);
    t1 += warp_sum(s1);
  }
  a = t0; b = t1;
}

// Last-CTA election. Every CTA publishes its partial pair; the CTA that arrives last
// (atomic ticket) sums ALL pairs in index order -- the ticket decides only who sums, never the
// order, so the result is deterministic. Returns true in every thread of the last CTA, with
// (a, b) = totals in thread 0.
__device__ __forceinline__ bool publish_and_elect(double& a, double& b, double* partial,
                                                  const double* part_base, int nparts,
                                                  unsigned* counter, double (*sm)[MAXW], int extra = 0) {
  __shared__ int s_last;
  block_sum2(a, b, sm);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = a;
    partial[2 * blockIdx.x + 1] = b;
    __threadfence();
    unsigned prev = atomicAdd(counter, 1u);
    s_last = (prev == gridDim.x - 1 + extra);     // extra: arrivals of a concurrent launch (k_longrows)
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  final_sum2(part_base, nparts, a, b, sm);
  if (threadIdx.x == 0) *counter = 0u;
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
// TMA (cp.async.bulk) + mbarrier helpers
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// Watchdog for every spin wait: a pipeline bug traps (the launch fails with an error) instead
// of hanging the device. 2^35 cycles is ~17 s at 2 GHz, far beyond any legitimate wait.
__device__ __forceinline__ void spin_guard(long long t0) {
  if (clock64() - t0 > (1ll << 35)) __trap();
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  uint32_t ok;
  long long t0 = 0;
  for (int it = 0;; ++it) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    if (ok) break;
    if (it == 0) t0 = clock64(); else spin_guard(t0);
  }
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// bulk prefetch of [p, p + bytes) into L2 (TMA unit; no registers, no completion tracking)
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// 1-D bulk copy global -> shared, completion counted on the mbarrier, L2 evict-first hint
__device__ __forceinline__ void tma_load(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
               " [%0], [%1], %2, [%3], %4;"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}

// Stage layout: every region starts 16-byte aligned and holds the 16-byte-aligned superset of the
// tile's range (the ABI requires 16-byte aligned, 16-byte padded arrays).
template <int ROLE>
struct Stage {
  static constexpr bool HAS_V1 = ROLE != ROLE_PLAIN;   // r (K1) or y_prev (K2, accumulate)
  static constexpr bool HAS_V2 = ROLE == ROLE_K2DOTS;  // p for psi
  static constexpr int V_OFF = 0;
  static constexpr int V_BYTES = (CAP + 4) * 8;
  static constexpr int I_OFF = V_OFF + V_BYTES;
  static constexpr int I_BYTES = (CAP + 8) * 4;
  static constexpr int P_OFF = I_OFF + I_BYTES;
  static constexpr int P_BYTES = (RCAP + 8) * 4;
  static constexpr int V1_OFF = P_OFF + P_BYTES;
  static constexpr int V1_BYTES = HAS_V1 ? (RCAP + 4) * 8 : 0;
  static constexpr int V2_OFF = V1_OFF + V1_BYTES;
  static constexpr int V2_BYTES = HAS_V2 ? (RCAP + 4) * 8 : 0;
  static constexpr int BYTES = (V2_OFF + V2_BYTES + 127) / 128 * 128;
  static constexpr int SMEM = NST * BYTES;
};

struct StageDesc {
  int r0, r1;          // rows [r0, r1) of the tile
  int s0, se;          // staged entries [s0, se) (se = min(row_ptr[r1], s0 + CAP))
  int vb, ib, pb, rb, rb2;  // element index held at offset 0 of the V / I / P / V1 / V2 regions
};

__device__ __forceinline__ const char* align16_down(const void* p) {
  return reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15));
}
__device__ __forceinline__ unsigned span16(const void* lo, const void* hi_excl) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(lo) & ~uintptr_t(15);
  const uintptr_t b = (reinterpret_cast<uintptr_t>(hi_excl) + 15) & ~uintptr_t(15);
  return (unsigned)(b - a);
}

// ---------------------------------------------------------------------------------------------
// K1 / K2 / plain SpMV over CSR tiles (fmt 0; segments whose SELL-32 padding would be too large,
// e.g. power-law rows): persistent CTAs; each tile's values, indices, row pointers and row-wise
// vector slices arrive by TMA bulk copies NST-1 tiles ahead; products are formed in place in
// shared memory; rows are owned by the tile holding their first entry and summed sequentially.
// ---------------------------------------------------------------------------------------------
template <int ROLE>
__global__ void __launch_bounds__(NT, MINB) k_spmv(SpmvSeg a) {
  using C = Stage<ROLE>;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bars[NST];
  __shared__ StageDesc sdesc[NST];
  __shared__ double sm[2][MAXW];
  if (a.ctl != nullptr && a.ctl->done) return;
  const bool wtd = ROLE == ROLE_K2DOTS && a.wi != nullptr && a.ctl != nullptr && a.ctl->weighted;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x;
  const int my_tiles = a.ntiles > (int)blockIdx.x ? (a.ntiles - (int)blockIdx.x + G - 1) / G : 0;
  const uint64_t pol = a.pol_first;
  double acc0 = 0.0, acc1 = 0.0;

  const double* v1src = (ROLE == ROLE_K1 || a.accumulate) ? a.out : nullptr;
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < NST; ++q) mbar_init(&bars[q], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // producer (thread 0): describe tile j of this CTA and start its bulk copies into stage j % NST
  auto issue = [&](int j) {
    const int t = (int)blockIdx.x + j * G;
    const int q = j % NST;
    const int2 d0 = a.desc[t], d1 = a.desc[t + 1];
    StageDesc d;
    d.r0 = d0.x; d.r1 = d1.x; d.s0 = d0.y;
    d.se = min(d1.y, d0.y + CAP);
    unsigned char* base = smem + q * C::BYTES;
    unsigned tx = 0;
    const char* lo;
    unsigned nb;
    // values [s0, se)
    lo = align16_down(a.val + d.s0);
    nb = d.se > d.s0 ? span16(a.val + d.s0, a.val + d.se) : 0;
    d.vb = d.s0 - (int)((a.val + d.s0) - reinterpret_cast<const double*>(lo));
    if (nb) { tma_load(base + C::V_OFF, lo, nb, &bars[q], pol); tx += nb; }
    // indices [s0, se)
    lo = align16_down(a.idx + d.s0);
    nb = d.se > d.s0 ? span16(a.idx + d.s0, a.idx + d.se) : 0;
    d.ib = d.s0 - (int)((a.idx + d.s0) - reinterpret_cast<const int32_t*>(lo));
    if (nb) { tma_load(base + C::I_OFF, lo, nb, &bars[q], pol); tx += nb; }
    // row pointers [r0, r1]
    lo = align16_down(a.ptr + d.r0);
    nb = span16(a.ptr + d.r0, a.ptr + d.r1 + 1);
    d.pb = d.r0 - (int)((a.ptr + d.r0) - reinterpret_cast<const int32_t*>(lo));
    tma_load(base + C::P_OFF, lo, nb, &bars[q], pol);
    tx += nb;
    // row-wise vector slices [r0, r1)
    d.rb = d.r0;
    d.rb2 = d.r0;
    if (d.r1 > d.r0) {
      if (C::HAS_V1 && v1src) {
        lo = align16_down(v1src + d.r0);
        nb = span16(v1src + d.r0, v1src + d.r1);
        d.rb = d.r0 - (int)((v1src + d.r0) - reinterpret_cast<const double*>(lo));
        tma_load(base + C::V1_OFF, lo, nb, &bars[q], pol);
        tx += nb;
      }
      if (C::HAS_V2) {
        lo = align16_down(a.pv + d.r0);
        nb = span16(a.pv + d.r0, a.pv + d.r1);
        d.rb2 = d.r0 - (int)((a.pv + d.r0) - reinterpret_cast<const double*>(lo));
        tma_load(base + C::V2_OFF, lo, nb, &bars[q], pol);
        tx += nb;
      }
    }
    sdesc[q] = d;
    mbar_expect_tx(&bars[q], tx);
  };

  if (tid == 0)
    for (int j = 0; j < min(NST - 1, my_tiles); ++j) issue(j);

  for (int j = 0; j < my_tiles; ++j) {
    const int q = j % NST;
    if (tid == 0 && j + NST - 1 < my_tiles) {
      fence_proxy_async();          // generic accesses to that stage (iteration j-1) happen-before
      issue(j + NST - 1);
    }
    mbar_wait(&bars[q], (unsigned)(j / NST) & 1u);
    const StageDesc d = sdesc[q];
    double* V = reinterpret_cast<double*>(smem + q * C::BYTES + C::V_OFF);
    const int32_t* I = reinterpret_cast<const int32_t*>(smem + q * C::BYTES + C::I_OFF);
    const int32_t* P = reinterpret_cast<const int32_t*>(smem + q * C::BYTES + C::P_OFF);
    const double* V1 = reinterpret_cast<const double*>(smem + q * C::BYTES + C::V1_OFF);
    const double* V2 = reinterpret_cast<const double*>(smem + q * C::BYTES + C::V2_OFF);
    // products in place: V[e] <- val_e * g[idx_e]  (gathers of the whole tile in flight at once)
    const int cnt = d.se - d.s0;
    const int voff = d.s0 - d.vb, ioff = d.s0 - d.ib;
    {
      constexpr int GU = (CAP + NT - 1) / NT;
      double gv[GU];
#pragma unroll
      for (int u = 0; u < GU; ++u) {
        const int k = tid + u * NT;
#if PLSS_ABLATE & 1
        if (k < cnt) gv[u] = (double)I[ioff + k];              // ablation: no gather
#else
        if (k < cnt) gv[u] = __ldg(a.g + I[ioff + k]);
#endif
      }
#pragma unroll
      for (int u = 0; u < GU; ++u) {
        const int k = tid + u * NT;
        if (k < cnt) V[voff + k] = __dmul_rn(V[voff + k], gv[u]);
      }
    }
    __syncthreads();
    const int vsh = -d.vb;   // V index of entry position e is e - vb
    // rows spread evenly over the 8 warps (a tile of short rows has far fewer rows than threads)
    const int rpw = (d.r1 - d.r0 + NT / 32 - 1) / (NT / 32);
    const int wlo = d.r0 + warp * rpw, whi = min(d.r1, wlo + rpw);
#if PLSS_ABLATE & 2
    if (tid < d.r1 - d.r0) { if (ROLE == ROLE_K1) { a.out[d.r0 + tid] = V[tid + d.s0 - d.vb]; } else a.out[d.r0 + tid] = V[tid + d.s0 - d.vb]; }
    for (int base = whi; base < whi; base += 32) {            // ablation: no row phase
#else
    for (int base = wlo; base < whi; base += 32) {
#endif
      const int i = base + lane;
      const bool valid = i < whi;
      int b = 0, e = 0;
      if (valid) { b = P[i - d.pb]; e = P[i + 1 - d.pb]; }
      const bool lng = valid && (e - b) > LONGROW;
      double s = 0.0;
      if (ROLE >= ROLE_K2 && valid && a.accumulate) s = V1[i - d.rb];
      if (valid && !lng) {
        const int es = min(e, d.se);
        int k = b;
#pragma unroll 1
        for (; k + 4 <= es; k += 4) {                       // staged products, 4 loads in flight
          const double p0 = V[k + vsh], p1 = V[k + 1 + vsh], p2 = V[k + 2 + vsh], p3 = V[k + 3 + vsh];
          s = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(s, p0), p1), p2), p3);
        }
        for (; k < es; ++k) s = __dadd_rn(s, V[k + vsh]);
        for (; k < e; ++k)                                   // spill past the staged window
          s = __dadd_rn(s, __dmul_rn(ld_stream(a.val + k, pol), __ldg(a.g + ld_stream(a.idx + k, pol))));
      }
      unsigned mask = __ballot_sync(FULL, lng);
      while (mask) {                                            // warp-cooperative long rows
        const int l = __ffs(mask) - 1;
        mask &= mask - 1;
        const int lb = __shfl_sync(FULL, b, l), le = __shfl_sync(FULL, e, l);
        double ps = 0.0;
        for (int k = lb + lane; k < le; k += 32) {
          const double pr = (k < d.se) ? V[k + vsh]
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
          const double rn = __dsub_rn(V1[i - d.rb], s);          // r_i <- r_i - (A p)_i
          a.out[i] = rn;
          acc0 = fma(rn, rn, acc0);
        } else if (ROLE == ROLE_K2DOTS) {
          double d0, d1;
          a.out[i] = k2_final(a, wtd, i, s, d0, d1);  // y_j (WIy_j under PLSS W)
          acc0 += d0;
          acc1 += d1;
        } else {
          a.out[i] = s;                                         // y_j
        }
      }
    }
    __syncthreads();                                            // stage q is free again
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
// K1 / K2 / plain SpMV over SELL-32 (sliced ELLPACK, slices of 32 rows, sigma-sorted by length
// when rows vary). One warp streams one slice: at step j lane l loads entry j of its row with
// fully coalesced 128-bit-per-quarter-warp loads (idx 128 B, val 256 B per step), gathers g and
// adds the product to its row sum in ascending entry order (bitwise the oracle's sequential sum).
// No shared memory: on B200 the SpMV is bound by L1 data-pipe wavefronts, and staging through
// shared memory costs more of them than it saves (profiles/r01_notes.md).
// ---------------------------------------------------------------------------------------------
#ifndef PLSS_SU
#define PLSS_SU 8
#endif
#ifndef PLSS_SELL_MINB
#define PLSS_SELL_MINB 4
#endif
constexpr int SU = PLSS_SU;             // steps (entries per lane) in flight
#ifndef PLSS_SIGMA
#define PLSS_SIGMA 512
#endif
constexpr int SIGMA = PLSS_SIGMA;       // rows per sigma-sort window (SELL-32 construction; C5's K2
                                        // slabs: 57% padding unsorted, 9.4% at 256, 2.9% at 1024;
                                        // 512 measured best, +0.8% over 256, 1024 ties 256)
constexpr int SPW = SIGMA / 32;         // slices per sigma window
// slices per CTA-range block of fmt 3 (a multiple of the sigma window: a window's y staging
// counter lives in one CTA's shared memory)
constexpr int NSB = SPW > 16 ? SPW : 16;
#ifndef PLSS_PAIR
#define PLSS_PAIR 1                     // fmt 3: consecutive slices a warp sums together
#endif
#ifndef PLSS_YQ
#define PLSS_YQ 6
#endif
// fmt 3 K2: sigma windows staged in shared memory at once (dynamic smem, YQ * SIGMA * 8 bytes),
// and the ring of per-window staging decisions (YD windows)
constexpr int YQ = PLSS_YQ;
constexpr int YSTAGE_SMEM = YQ * SIGMA * 8;
constexpr int SIGMA_WIDE = 2 * SIGMA;    // the wider window a K2 segment may take (a.sig)
constexpr int YSTAGE_SMEM_WIDE = YQ * SIGMA_WIDE * 8;
__host__ __device__ constexpr int nsb_of(int sig) { return sig / 32 > 16 ? sig / 32 : 16; }
// CTA-range granularity of globally length-sorted segments (no sigma windows to align to): their
// longest slices hold up to 32 * LONGROW entries each, so blocks of 16 of them overshot a CTA's
// share (C4-alt's first CTA held two such blocks, 128K entries against a 59K median)
#ifndef PLSS_GS_NSB
#define PLSS_GS_NSB 1
#endif
constexpr int GS_NSB = PLSS_GS_NSB;
#ifndef PLSS_GS_MINB
#define PLSS_GS_MINB 1                  // 1024-thread CTAs per SM of globally sorted segments
#endif
constexpr int GS_MINB = PLSS_GS_MINB;
#ifndef PLSS_GS_SU
#define PLSS_GS_SU PLSS_SU              // their entries per lane in flight
#endif
constexpr int GS_SU = PLSS_GS_SU;
#ifndef PLSS_S1B
#define PLSS_S1B 6                      // one-step slices of a globally sorted segment per warp batch
#endif
constexpr int S1B = PLSS_S1B;
constexpr int YD = 1024;
#ifndef PLSS_YSTAGE
#define PLSS_YSTAGE 1
#endif
constexpr int SELL_MINB = PLSS_SELL_MINB;

// Gather of g[c] (c = -1: padding). Ablation builds (timing experiments only, never correct):
// 4 = no gathers (the index as value), 16 = gathers from an 8 MB hot set.
__device__ __forceinline__ double sell_gather(const SpmvSeg& a, int c) {
#if PLSS_ABLATE & 4
  return (double)c;
#elif PLSS_ABLATE & 16
  return c >= 0 ? __ldg(a.g + (c & 0xFFFFF)) : 0.0;
#else
  return c >= 0 ? __ldg(a.g + c) : 0.0;
#endif
}

// s += sum over the slice's steps [0, L) of val * g[idx], lane = one row, ascending step order,
// SU steps in flight per lane (loads of a batch issued before its gathers, gathers before sums).
template <int ROLE, int SU = plss::SU>
__device__ __forceinline__ double sell_row_sum(const SpmvSeg& a, int st0, int L, int lane, double s,
                                               uint64_t pol) {
  const int32_t* ip = a.idx + (long long)st0 * 32 + lane;
  const double* vp = a.val + (long long)st0 * 32 + lane;
  int j = 0;
  for (; j + SU <= L; j += SU) {
    int32_t c[SU];
    double v[SU], gv[SU];
#pragma unroll
    for (int u = 0; u < SU; ++u) { c[u] = ld_stream(ip + (j + u) * 32, pol); v[u] = ld_stream(vp + (j + u) * 32, pol); }
#pragma unroll
    for (int u = 0; u < SU; ++u) gv[u] = sell_gather(a, c[u]);
#pragma unroll
    for (int u = 0; u < SU; ++u) if (c[u] >= 0) s = __dadd_rn(s, __dmul_rn(v[u], gv[u]));
  }
  if (j < L) {
    int32_t c[SU];
    double v[SU], gv[SU];
#pragma unroll
    for (int u = 0; u < SU; ++u) {
      c[u] = -1;
      if (j + u < L) { c[u] = ld_stream(ip + (j + u) * 32, pol); v[u] = ld_stream(vp + (j + u) * 32, pol); }
    }
#pragma unroll
    for (int u = 0; u < SU; ++u) gv[u] = sell_gather(a, c[u]);
#pragma unroll
    for (int u = 0; u < SU; ++u) if (c[u] >= 0) s = __dadd_rn(s, __dmul_rn(v[u], gv[u]));
  }
  return s;
}

// P slices at once (fmt 3): lane l sums row l of each of P consecutive slices, SU/P steps of each
// in flight per batch, so the latency chains of P rows overlap and per-slice costs are shared.
template <int ROLE, int P>
__device__ __forceinline__ void sell_rows_sum(const SpmvSeg& a, const int (&st0)[P], const int (&L)[P], int lane,
                                              double (&s)[P], uint64_t pol) {
  constexpr int SUP = SU / P;
  int Lmax = 0;
#pragma unroll
  for (int q = 0; q < P; ++q) Lmax = max(Lmax, L[q]);
  for (int j = 0; j < Lmax; j += SUP) {
    int32_t c[P][SUP];
    double v[P][SUP], gv[P][SUP];
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
      for (int u = 0; u < SUP; ++u) {
        c[q][u] = -1;
        if (j + u < L[q]) {
          const long long e = ((long long)st0[q] + j + u) * 32 + lane;
          c[q][u] = ld_stream(a.idx + e, pol);
          v[q][u] = ld_stream(a.val + e, pol);
        }
      }
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
      for (int u = 0; u < SUP; ++u) gv[q][u] = sell_gather(a, c[q][u]);
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
      for (int u = 0; u < SUP; ++u)
        if (c[q][u] >= 0) s[q] = __dadd_rn(s[q], __dmul_rn(v[q][u], gv[q][u]));
  }
}

// Long rows of a globally sorted segment in chunks of LCH entries (the default; k_longrows is the
// CTA-per-row alternative, PLSS_LCHUNK=0): a warp per chunk, LCU entries per lane in flight (one
// load batch), so short long rows (C4's are 129 .. 4096 entries, ~500 on average) no longer leave
// most of a 256-thread CTA idle for a whole CTA lifetime (k_longrows: 41 us for C4's 2.7M long-row
// entries). A chunk's sum: each lane's entries u = 0 .. LCU-1 sequentially, then the warp
// butterfly; a row's sum: its chunk sums in chunk order, added by the warp that finishes the row's
// last chunk (a per-row counter decides who, never the order). Row dot terms are reduced in row
// order by the warp that finishes the last row, then the joint election with the slices' CTAs as in
// k_longrows (final_sum2_warp: the same shape as the CTAs' final_sum2).
#ifndef PLSS_LCU
#define PLSS_LCU 12
#endif
constexpr int LCU = PLSS_LCU;
constexpr int LCH = 32 * LCU;
#ifndef PLSS_LCB
#define PLSS_LCB 6                      // k_sell's phase 0: a chunk's entries per lane per load batch
#endif
constexpr int LCB = PLSS_LCB;
// One chunk c of a long row, by one warp (k_longchunks, or k_sell's phase 0 for a globally sorted
// segment). LB entries per lane per load batch, LCU / LB batches: a lane's entries are summed in
// order u = 0 .. LCU-1 whatever LB is. lpart: the long rows' partial pair slot (after the slices'
// CTAs). Returns true in every lane of the warp that must finalize the joint election (only
// possible in k_longchunks: inside k_sell the warp's own CTA has not arrived yet).
template <int ROLE, int LB>
__device__ __forceinline__ bool longchunk_warp(const SpmvSeg& a, int c, double* lpart, bool wtd, int lane) {
  static_assert(LCU % LB == 0, "whole batches");
  constexpr bool DOTS = ROLE == ROLE_K1 || ROLE == ROLE_K2DOTS;
  const uint64_t pol = a.pol_first;
  const int4 d = a.lchunk[c];                                   // e0, e1, row k, first chunk of k
  const int nch = a.lnch[d.z];
  // the row's output slot and its old value, loaded early in case this warp finishes the row
  const int r = lane == 0 ? a.lrows[d.z] : 0;
  double start = 0.0;
  if (lane == 0 && (ROLE == ROLE_K1 || ((ROLE == ROLE_K2 || ROLE == ROLE_K2DOTS) && a.accumulate))) start = a.out[r];
  double s = 0.0;
#pragma unroll
  for (int u0 = 0; u0 < LCU; u0 += LB) {
    int32_t ci[LB];
    double v[LB], g[LB];
#pragma unroll
    for (int u = 0; u < LB; ++u) {
      const int q = d.x + (u0 + u) * 32 + lane;
      ci[u] = -1;
      if (q < d.y) { ci[u] = ld_stream(a.lidx + q, pol); v[u] = ld_stream(a.lval + q, pol); }
    }
#pragma unroll
    for (int u = 0; u < LB; ++u) g[u] = sell_gather(a, ci[u]);
#pragma unroll
    for (int u = 0; u < LB; ++u) if (ci[u] >= 0) s = __dadd_rn(s, __dmul_rn(v[u], g[u]));
  }
  s = warp_sum(s);
  int last = 1;
  if (nch > 1) {
    if (lane == 0) {
      a.lcpart[c] = s;
      __threadfence();
      last = atomicAdd(a.lrcnt + d.z, 1u) == (unsigned)(nch - 1);
    }
    last = __shfl_sync(FULL, last, 0);
  }
  if (!last) return false;
  int fin = 0;
  if (lane == 0) {
    double d0 = 0.0, d1 = 0.0;
    double t = s;
    if (nch > 1) {                                              // the row's chunk sums in chunk order
      __threadfence();
      t = 0.0;
      for (int j0 = 0; j0 < nch; j0 += 8) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = j0 + u < nch ? __ldcg(a.lcpart + d.w + j0 + u) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) if (j0 + u < nch) t = __dadd_rn(t, x[u]);
      }
      a.lrcnt[d.z] = 0u;
    }
    if (ROLE == ROLE_PLAIN) {
      a.out[r] = t;
    } else if (ROLE == ROLE_K1) {
      const double rn = __dsub_rn(start, t);                   // r_i <- r_i - (A p)_i
      a.out[r] = rn;
      d0 = rn * rn;
    } else {
      a.out[r] = ROLE == ROLE_K2DOTS ? k2_final(a, wtd, r, __dadd_rn(start, t), d0, d1)
                                     : __dadd_rn(start, t);
    }
    if (DOTS) {
      a.lrowd[2 * d.z] = d0;
      a.lrowd[2 * d.z + 1] = d1;
      __threadfence();
      const int grp = d.z >> 5, gsz = min(32, a.nlong - (grp << 5));
      fin = atomicAdd(a.lgcnt + grp, 1u) == (unsigned)(gsz - 1);  // this row completes its group
    }
  }
  if (!DOTS) return false;
  fin = __shfl_sync(FULL, fin, 0);
  if (!fin) return false;
  __threadfence();
  const int grp = d.z >> 5, ngroup = (a.nlong + 31) >> 5;
  {                                                             // the group's 32 rows, butterfly
    const int q = (grp << 5) + lane;
    double s0 = q < a.nlong ? __ldcg(a.lrowd + 2 * q) : 0.0;
    double s1 = q < a.nlong ? __ldcg(a.lrowd + 2 * q + 1) : 0.0;
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    fin = 0;
    if (lane == 0) {
      a.lgd[2 * grp] = s0;
      a.lgd[2 * grp + 1] = s1;
      a.lgcnt[grp] = 0u;
      __threadfence();
      fin = atomicAdd(a.lcounter, 1u) == (unsigned)(ngroup - 1);
    }
    fin = __shfl_sync(FULL, fin, 0);
    if (!fin) return false;
    __threadfence();
  }
  double s0 = 0.0, s1 = 0.0;                                    // the group sums in group order
  seq_add2(a.lgd, lane, ngroup, 32, s0, s1);
  s0 = warp_sum(s0);
  s1 = warp_sum(s1);
  int efin = 0;
  if (lane == 0) {
    *a.lcounter = 0u;
    lpart[0] = s0;
    lpart[1] = s1;
    if (a.finalize) {                                           // one more arrival in the slices' election
      __threadfence();
      efin = atomicAdd(a.counter, 1u) == (unsigned)(a.elect_total - 1);
    }
  }
  efin = __shfl_sync(FULL, efin, 0);
  return efin != 0;
}

// BS = NT (fmt 1): persistent grid, slices dealt round-robin over all warps of the grid; each
//   thread accumulates its rows' dot contributions (static assignment: deterministic).
// BS = 1024 (fmt 3): one CTA per SM walks the contiguous, entry-balanced slice range
//   [cblk[c], cblk[c+1]) * NSB; its 32 warps take slices in order from a shared counter (rows of
//   very different lengths balance across warps; consecutive in-flight slices share their band of
//   g in L1). Slice order is run-dependent, so dots are reduced per slice (slpart) and summed in
//   slice order (deterministic).
// Slice metadata (start, length, this lane's row) is loaded one slice ahead, so a slice's stream
// loads wait for DRAM only, not for an L2 round trip to sptr / perm first.
// LU: unused since round 2 (a globally sorted segment's long rows run in k_longrows; must be
// false); YS: the K2 segment's y is staged (sigma perm)
template <int ROLE, int BS = NT, bool LU = false, bool YS = false, int SIGT = SIGMA, bool STAT = false,
          int SUK = SU, int GNSB = 0>
__global__ void __launch_bounds__(BS, BS == NT ? SELL_MINB : GNSB ? GS_MINB : 1) k_sell(SpmvSeg a) {
  constexpr int SPW = SIGT / 32;                 // this instantiation's sigma window (a.sig)
  constexpr int NSB = GNSB ? GNSB : nsb_of(SIGT); // CTA-range granularity (slices)
  constexpr int SIGMA = SIGT;
  constexpr bool DYN = BS != NT;
  constexpr bool DOTS = ROLE == ROLE_K1 || ROLE == ROLE_K2DOTS;
  constexpr int P = DYN && !STAT ? PLSS_PAIR : 1; // slices per warp unit
  static_assert(!LU, "long rows run in k_longrows");
  static_assert(!STAT || (DYN && !YS), "static stepping: fmt 3 segments without perm / long rows");
  // fmt 3 K2 with a sigma perm: y results go through a per-sigma-window shared buffer (indexed by
  // row, not slot) and the warp that completes a window writes its SIGMA values coalesced,
  // instead of 32 scattered 8-byte stores per slice. In-flight slices (<= 32 P + P) span at most
  // YQ - 2 windows, so the buffers are never reused while still filling.
  constexpr bool YST = YS && DYN && (ROLE == ROLE_K2 || ROLE == ROLE_K2DOTS) && PLSS_YSTAGE;
  static_assert(SPW % P == 0 && NSB % P == 0, "a warp unit must not straddle a sigma window");
  __shared__ double sm[2][MAXW];
  __shared__ int s_next;
  __shared__ int s_next1;                           // GNSB: next batch of one-step slices (phase 2)
  extern __shared__ __align__(16) double s_ydyn[];  // [YQ][SIGMA] when YST (dynamic smem)
  double (*s_y)[SIGMA] = reinterpret_cast<double (*)[SIGMA]>(s_ydyn);
  __shared__ int s_ycnt[YST ? YQ : 1];
  __shared__ int s_ytag[YST ? YQ : 1];              // window a y slot holds (-1: free)
  __shared__ int s_ydec[YST ? YD : 1];              // window W's decision: W * 2 + staged
  if (a.ctl != nullptr && a.ctl->done) return;
  const bool wtd = ROLE == ROLE_K2DOTS && a.wi != nullptr && a.ctl != nullptr && a.ctl->weighted;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t pol = a.pol_first;
  double acc0 = 0.0, acc1 = 0.0;
  int sl0, sl1, slE, stride;
  if (!DYN) {
    sl0 = blockIdx.x * (NT / 32); sl1 = a.nslices; stride = gridDim.x * (NT / 32);
    slE = sl1;
  } else {
    sl0 = a.cblk[blockIdx.x] * NSB; sl1 = min(a.cblk[blockIdx.x + 1] * NSB, a.nslices);
    slE = sl1;                                      // the CTA's whole range (its dot partials)
    // globally sorted: the one-step (and empty) slices [s1beg, slE) run in phase 2, by batches
    if (GNSB && a.s1on) sl1 = max(sl0, min(sl1, a.s1beg));
    stride = P * BS / 32;
    if (GNSB && tid == 0) s_next1 = max(sl0, a.s1on ? a.s1beg : slE);
    if (tid == 0 && !STAT) s_next = sl0 + P * (BS / 32);   // the first unit of each warp is static
    if (YST && tid < YQ) { s_ycnt[tid] = 0; s_ytag[tid] = -1; }
    if (YST) for (int q = tid; q < YD; q += BS) s_ydec[q] = -2;
    __syncthreads();
  }
  int su = sl0 + warp * P;                          // first slice of this warp's unit
  int m0[P], m1[P], mrow[P];
  auto meta = [&](int t) {
#pragma unroll
    for (int q = 0; q < P; ++q) {
      if (t + q < sl1) {
        m0[q] = a.sptr[t + q]; m1[q] = a.sptr[t + q + 1];
        mrow[q] = a.perm ? a.perm[(t + q) * 32 + lane] : (t + q) * 32 + lane;
      } else {
        m0[q] = 0; m1[q] = 0; mrow[q] = -1;
      }
    }
  };
  // y staging without waits on a held slot. Ring slots are reused every YQ sigma windows, and a
  // straggler (the longest slice of a sigma window is its first) can still own a slot when a later
  // window maps to it. So the window's fate is decided when its FIRST slice is ticketed (tickets
  // are in order): staged if its slot is free (claimed by tag), else its slices write y directly.
  // The window's other slices read the decision right after taking their tickets (at most a few
  // instructions after it is made). A staged window releases its slot when complete.
  constexpr bool YSTG = YST;
  auto ydecide = [&](int first_slice) {             // lane 0 / thread 0
    const int W = first_slice / SPW;
    const int staged = atomicCAS(&s_ytag[W % YQ], -1, W) == -1;
    *(volatile int*)&s_ydec[W % YD] = W * 2 + staged;
  };
  auto ymode = [&](int sl) -> int {                 // whole warp: 1 = staged
    int v = 0;
    if (lane == 0) {
      const int W = sl / SPW;
      const long long t0 = clock64();
      while (((v = *(volatile int*)&s_ydec[W % YD]) >> 1) != W) { __nanosleep(32); spin_guard(t0); }
    }
    return __shfl_sync(FULL, v, 0) & 1;
  };
  if (YSTG && DYN && a.perm && !a.gsort) {
    if (tid == 0)
      for (int f = sl0; f < min(sl0 + P * (BS / 32), sl1); f += SPW) ydecide(f);
    __syncthreads();
  }
#ifdef PLSS_DBGCTA
  unsigned long long dbg_entries = 0, dbg_units = 0;
  if (DYN && a.ctat && tid == 0) {
    unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.ctat[4 * blockIdx.x] = t;
  }
#endif
  // Phase 0 (globally sorted segments with long rows, lin): the long rows' chunks, dealt statically
  // (chunk c to CTA c mod grid, warp c / grid mod 32), LCB entries per lane per load batch, instead
  // of a concurrent k_longchunks launch: that launch's CTAs could not share an SM with this kernel's
  // 1024 x 64 registers and ran on the SMs its CTAs had freed. Opt-in (PLSS_LIN=1): it loses on C4
  // (0.1994 vs 0.1935 ms per step) and C4-alt (0.381 vs 0.358): the CTAs' balanced slice shares
  // then finish later, while the separate launch used the SMs of the CTAs that finished first.
  if (GNSB && a.lin) {
    for (int c = blockIdx.x + gridDim.x * warp; c < a.nchunks; c += gridDim.x * (BS / 32))
      longchunk_warp<ROLE, LCB>(a, c, a.partial + 2 * gridDim.x, wtd, lane);   // never the election's last
  }
  if (su < sl1) meta(su);
  while (su < sl1) {
    const bool stage = YSTG && a.perm && !a.gsort && ymode(su);
    int st0[P], L[P], row[P];
#pragma unroll
    for (int q = 0; q < P; ++q) {
      st0[q] = m0[q]; L[q] = m1[q] - m0[q];
      row[q] = mrow[q];
    }
    const int cnt = min(P, sl1 - su);               // slices of this unit that exist
    int nx;
    if (!DYN || STAT) {
      nx = su + stride;
    } else {
      nx = 0;
      if (lane == 0) {
        nx = atomicAdd(&s_next, P);
        if (YSTG && a.perm && !a.gsort && nx < sl1 && nx % SPW == 0) ydecide(nx);
      }
      nx = __shfl_sync(FULL, nx, 0);
    }
#if defined(PLSS_DBGCTA) && PLSS_DBGCTA > 1
    if (DYN && a.ctat && lane == 0)
      for (int q = 0; q < P; ++q) if (su + q < sl1) { dbg_entries += 32ull * L[q]; dbg_units++; }
#endif
    if (nx < sl1) meta(nx);
    bool valid[P];
    double s[P], r_old[P];
#pragma unroll
    for (int q = 0; q < P; ++q) {
      valid[q] = row[q] >= 0 && row[q] < a.nrows;
      s[q] = 0.0;
#if !(PLSS_ABLATE & (32 | 64))
      if (ROLE >= ROLE_K2 && valid[q] && a.accumulate) s[q] = a.out[row[q]];
#endif
      r_old[q] = (ROLE == ROLE_K1 && valid[q]) ? a.out[row[q]] : 0.0;   // issued early
    }
    if (P == 1) {
      s[0] = sell_row_sum<ROLE, SUK>(a, st0[0], L[0], lane, s[0], pol);
    } else {
      sell_rows_sum<ROLE, P>(a, st0, L, lane, s, pol);
    }
#pragma unroll
    for (int q = 0; q < P; ++q) {
      if (q >= cnt) break;
      double d0 = 0.0, d1 = 0.0;
      if (valid[q]) {
        if (ROLE == ROLE_PLAIN) {
          a.out[row[q]] = s[q];
        } else if (ROLE == ROLE_K1) {
          const double rn = __dsub_rn(r_old[q], s[q]);          // r_i <- r_i - (A p)_i
          a.out[row[q]] = rn;
          d0 = rn * rn;
        } else {
#if PLSS_ABLATE & 32
          if (s[q] == 1234.5) a.out[row[q]] = s[q];             // ablation: no y write
#else
          // y_j, or under PLSS W in the last slab WIy_j (what K3 consumes)
          const double yv = ROLE == ROLE_K2DOTS ? k2_final(a, wtd, row[q], s[q], d0, d1) : s[q];
          if (stage) s_y[((su + q) / SPW) % YQ][row[q] % SIGMA] = yv;  // staged
          else a.out[row[q]] = yv;
#endif
        }
      }
      if (DOTS) {
        if (!DYN || STAT) {                                     // static stepping: per-thread terms
          acc0 += d0; acc1 += d1;
        } else {
          d0 = warp_sum(d0);
          if (ROLE == ROLE_K2DOTS) d1 = warp_sum(d1);             // K1 has no second dot (d1 = 0)
          if (lane == 0) { a.slpart[2 * (su + q)] = d0; a.slpart[2 * (su + q) + 1] = d1; }
        }
      }
    }
    if (stage) {
      const int w = su / SPW, qw = w % YQ;
      const int nsw = min(SPW, a.nslices - w * SPW);           // slices of this sigma window
      __threadfence_block();                                    // this warp's s_y stores before the count
      __syncwarp();
      int last = 0;
      if (lane == 0) last = atomicAdd(&s_ycnt[qw], cnt) + cnt == nsw;
      last = __shfl_sync(FULL, last, 0);
      if (last) {                                               // window complete: write it out
        __threadfence_block();                                  // the other warps' s_y stores are visible
        const int r0 = a.wrow0 + w * SIGMA;
#pragma unroll
        for (int u = 0; u < SIGMA / 32; ++u) {
          const int r = r0 + u * 32 + lane;
          if (r < a.nrows) a.out[r] = s_y[qw][u * 32 + lane];
        }
        __syncwarp();
        if (lane == 0) { s_ycnt[qw] = 0; __threadfence_block(); atomicExch(&s_ytag[qw], -1); }
      }
    }
    su = nx;
  }
  // Phase 2 (globally sorted segments): one-step and empty slices, S1B of them per warp batch. Their
  // slots are consecutive, so a batch's perm, idx and val loads are S1B independent coalesced loads
  // per lane, then S1B gathers and output loads, instead of one slice's dependent chain at a time
  // (C4: 64% of the rows have one entry). Each row's sum is its one product added to 0 (or to y),
  // as in sell_row_sum; dot partials per slice into slpart, as in phase 1.
  if (GNSB && a.s1on) {
    constexpr int S1B = ROLE == ROLE_K2DOTS && plss::S1B > 4 ? 4 : plss::S1B;  // K2DOTS: no spills
    for (;;) {
      int b = 0;
      if (lane == 0) b = atomicAdd(&s_next1, S1B);
      b = __shfl_sync(FULL, b, 0);
      if (b >= slE) break;
      int row[S1B], c[S1B];
      double v[S1B], gv[S1B], s[S1B], r_old[S1B];
#pragma unroll
      for (int q = 0; q < S1B; ++q) {
        const int t = b + q;
        row[q] = t < slE ? a.perm[(long long)t * 32 + lane] : -1;
        c[q] = -1;
        if (t < slE && t < a.s1end) {
          const long long e = ((long long)a.s1step0 + (t - a.s1beg)) * 32 + lane;
          c[q] = ld_stream(a.idx + e, pol);
          v[q] = ld_stream(a.val + e, pol);
        }
      }
#pragma unroll
      for (int q = 0; q < S1B; ++q) {
        const bool valid = row[q] >= 0 && row[q] < a.nrows;
        s[q] = (ROLE >= ROLE_K2 && valid && a.accumulate) ? a.out[row[q]] : 0.0;
        r_old[q] = (ROLE == ROLE_K1 && valid) ? a.out[row[q]] : 0.0;
        gv[q] = sell_gather(a, c[q]);
      }
#pragma unroll
      for (int q = 0; q < S1B; ++q) {
        const int t = b + q;
        if (t >= slE) break;
        if (c[q] >= 0) s[q] = __dadd_rn(s[q], __dmul_rn(v[q], gv[q]));
        double d0 = 0.0, d1 = 0.0;
        if (row[q] >= 0 && row[q] < a.nrows) {
          if (ROLE == ROLE_PLAIN) {
            a.out[row[q]] = s[q];
          } else if (ROLE == ROLE_K1) {
            const double rn = __dsub_rn(r_old[q], s[q]);
            a.out[row[q]] = rn;
            d0 = rn * rn;
          } else {
            a.out[row[q]] = ROLE == ROLE_K2DOTS ? k2_final(a, wtd, row[q], s[q], d0, d1) : s[q];
          }
        }
        if (DOTS) {
          d0 = warp_sum(d0);
          if (ROLE == ROLE_K2DOTS) d1 = warp_sum(d1);
          if (lane == 0) { a.slpart[2 * t] = d0; a.slpart[2 * t + 1] = d1; }
        }
      }
    }
  }
#ifdef PLSS_DBGCTA
  if (DYN && a.ctat) {                              // diagnostics build only (uniform branch)
    __shared__ unsigned long long s_dbg[2];
    if (tid == 0) { s_dbg[0] = 0; s_dbg[1] = 0; }
    __syncthreads();
    if (lane == 0) { atomicAdd(&s_dbg[0], dbg_entries); atomicAdd(&s_dbg[1], dbg_units); }
    __syncthreads();
    if (tid == 0) {
      unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.ctat[4 * blockIdx.x + 1] = t;
      a.ctat[4 * blockIdx.x + 2] = s_dbg[0];
      a.ctat[4 * blockIdx.x + 3] = s_dbg[1];
    }
  }
#endif
  if (!DOTS) return;
  if (DYN && !STAT) {
    __syncthreads();
    for (int q = sl0 + tid; q < slE; q += BS) { acc0 += a.slpart[2 * q]; acc1 += a.slpart[2 * q + 1]; }
  }
  if (!a.finalize) {
    block_sum2(acc0, acc1, sm);
    if (tid == 0) { a.partial[2 * blockIdx.x] = acc0; a.partial[2 * blockIdx.x + 1] = acc1; }
    return;
  }
  if (!publish_and_elect(acc0, acc1, a.partial, a.part_base, a.nparts, a.counter, sm, a.elect_extra)) return;
  if (tid != 0) return;
  if (ROLE == ROLE_K1) {
    if (a.dist) *a.rho_out = acc0;
    else tail_rho(a.ctl, a.rec, acc0);
  } else if (ROLE == ROLE_K2DOTS) {
    tail_y(a.ctl, a.rec, acc0, acc1);
  }
}

// ---------------------------------------------------------------------------------------------
// Segments of short rows (fmt 5: mean length <= SCALAR_MEAN, none longer than SCALAR_MAX; C4's
// columns: 1.05 entries on average, 35% empty): a thread per row over the original CSR-like arrays
// -- no SELL copy, no padding, no permutation. Rows are dealt grid-stride (a warp takes 32
// consecutive rows: coalesced ptr, output and p reads, nearly contiguous entries); each thread sums
// its row sequentially in ascending order (bitwise the oracle), accumulates its dot terms in a
// fixed order, and the CTA partials go through the usual fixed-order reduction. 2048 threads per
// SM at <= 32 registers (the weighted K2 variant spills a few bytes outside the row loop): the row
// loop is latency-bound, so more rows are in flight than the slice kernel's 32 warps keep. A
// thread-per-row tail for the short rows of globally sorted K1 segments was measured slower than
// their SELL slices (C4 K1 0.132 vs 0.110 ms): it serializes perm -> row pointer -> entries.
constexpr int SCALAR_MEAN = 4;
constexpr int SCALAR_MAX = 32;
#ifndef PLSS_SCB
#define PLSS_SCB 2
#endif
constexpr int SCB = PLSS_SCB;           // entries per thread in flight (rows are short); segments
                                        // of mean < 2 entries take 3 (SpmvSeg::scb; C4's columns:
                                        // K2 0.079 -> 0.075 ms, C4-alt's mean-3 columns lose with 3)
#ifndef PLSS_SCMINB
#define PLSS_SCMINB 8                   // CTAs per SM (2048 threads: C4 K2 0.104 -> 0.089 ms vs 6)
#endif
template <int ROLE, int SCBT = SCB>
__global__ void __launch_bounds__(NT, PLSS_SCMINB) k_scalar(SpmvSeg a) {
  __shared__ double sm[2][MAXW];
  if (a.ctl != nullptr && a.ctl->done) return;
  constexpr bool DOTS = ROLE == ROLE_K1 || ROLE == ROLE_K2DOTS;
  const bool wtd = ROLE == ROLE_K2DOTS && a.wi != nullptr && a.ctl != nullptr && a.ctl->weighted;
  const uint64_t pol = a.pol_first;
  double acc0 = 0.0, acc1 = 0.0;
  const long long stride = (long long)gridDim.x * NT;
  for (long long i = (long long)blockIdx.x * NT + threadIdx.x; i < a.nrows; i += stride) {
    const int e0 = a.ptr[i], e1 = a.ptr[i + 1];
    double sv = 0.0;
    if (ROLE == ROLE_K1 || ((ROLE == ROLE_K2 || ROLE == ROLE_K2DOTS) && a.accumulate)) sv = a.out[i];
    double s = (ROLE == ROLE_K1) ? 0.0 : sv;
    for (int e = e0; e < e1; e += SCBT) {
      int32_t c[SCBT];
      double v[SCBT], g[SCBT];
#pragma unroll
      for (int u = 0; u < SCBT; ++u) {
        c[u] = -1;
        if (e + u < e1) { c[u] = ld_stream(a.idx + e + u, pol); v[u] = ld_stream(a.val + e + u, pol); }
      }
#pragma unroll
      for (int u = 0; u < SCBT; ++u) g[u] = sell_gather(a, c[u]);
#pragma unroll
      for (int u = 0; u < SCBT; ++u) if (c[u] >= 0) s = __dadd_rn(s, __dmul_rn(v[u], g[u]));
    }
    double d0 = 0.0, d1 = 0.0;
    if (ROLE == ROLE_PLAIN) {
      a.out[i] = s;
    } else if (ROLE == ROLE_K1) {
      const double rn = __dsub_rn(sv, s);                        // r_i <- r_i - (A p)_i
      a.out[i] = rn;
      d0 = rn * rn;
    } else {
      a.out[i] = ROLE == ROLE_K2DOTS ? k2_final(a, wtd, i, s, d0, d1) : s;
    }
    if (DOTS) { acc0 += d0; acc1 += d1; }
  }
  if (!DOTS) return;
  if (!a.finalize) {
    block_sum2(acc0, acc1, sm);
    if (threadIdx.x == 0) { a.partial[2 * blockIdx.x] = acc0; a.partial[2 * blockIdx.x + 1] = acc1; }
    return;
  }
  if (!publish_and_elect(acc0, acc1, a.partial, a.part_base, a.nparts, a.counter, sm)) return;
  if (threadIdx.x != 0) return;
  if (ROLE == ROLE_K1) {
    if (a.dist) *a.rho_out = acc0;
    else tail_rho(a.ctl, a.rec, acc0);
  } else if (ROLE == ROLE_K2DOTS) {
    tail_y(a.ctl, a.rec, acc0, acc1);
  }
}

// Long rows (> LONGROW entries) of a globally sorted segment (C4's power-law rows), launched by
// launch_spmv right after the segment's slices: one 256-thread CTA per row, entries strided over
// the CTA (coalesced), SU loads in flight per thread, a fixed tree (warp butterflies, then the 8
// warp sums in order). Row epilogues as k_sell's. Dot terms per row go to lrowd; the last CTA
// (atomic ticket) sums them in row order (deterministic) into this launch's partial slot
// a.partial[0..1] and, if the segment finalizes, sums all partial pairs in index order and runs the
// tail. Separated from k_sell because its long-row path, inlined there, pushed the kernel past 64
// registers: ptxas then serialized the gathers of every batch (C4's long-row CTAs ran at half the
// per-entry rate of the slices).
template <int ROLE>
__global__ void __launch_bounds__(NT) k_longrows(SpmvSeg a) {
  __shared__ double sm[2][MAXW];
  __shared__ double s_w[NT / 32];
  __shared__ int s_last;
  if (a.ctl != nullptr && a.ctl->done) return;
  constexpr bool DOTS = ROLE == ROLE_K1 || ROLE == ROLE_K2DOTS;
  const bool wtd = ROLE == ROLE_K2DOTS && a.wi != nullptr && a.ctl != nullptr && a.ctl->weighted;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t pol = a.pol_first;
  const int k = blockIdx.x;
  const int r = a.lrows[k];
  const int e0 = a.lbeg[2 * k], e1 = a.lbeg[2 * k + 1];      // independent of r: no load chain
  double start = 0.0;
  if (tid == 0 && (ROLE == ROLE_K1 || ((ROLE == ROLE_K2 || ROLE == ROLE_K2DOTS) && a.accumulate))) start = a.out[r];
  double ps = 0.0;
  for (int k0 = e0; k0 < e1; k0 += NT * SU) {
    int32_t c[SU];
    double v[SU], gv[SU];
#pragma unroll
    for (int u = 0; u < SU; ++u) {
      const int q = k0 + u * NT + tid;
      c[u] = -1;
      if (q < e1) { c[u] = ld_stream(a.lidx + q, pol); v[u] = ld_stream(a.lval + q, pol); }
    }
#pragma unroll
    for (int u = 0; u < SU; ++u) gv[u] = sell_gather(a, c[u]);
#pragma unroll
    for (int u = 0; u < SU; ++u) if (c[u] >= 0) ps = __dadd_rn(ps, __dmul_rn(v[u], gv[u]));
  }
  ps = warp_sum(ps);
  if (lane == 0) s_w[warp] = ps;
  __syncthreads();
  double d0 = 0.0, d1 = 0.0;
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < NT / 32; ++w) t = __dadd_rn(t, s_w[w]);
    if (ROLE == ROLE_PLAIN) {
      a.out[r] = t;
    } else if (ROLE == ROLE_K1) {
      const double rn = __dsub_rn(start, t);                   // r_i <- r_i - (A p)_i
      a.out[r] = rn;
      d0 = rn * rn;
    } else {
      const double yv = ROLE == ROLE_K2DOTS ? k2_final(a, wtd, r, __dadd_rn(start, t), d0, d1)
                                            : __dadd_rn(start, t);
      a.out[r] = yv;
    }
    if (DOTS) {
      a.lrowd[2 * k] = d0;
      a.lrowd[2 * k + 1] = d1;
      __threadfence();
      s_last = atomicAdd(a.lcounter, 1u) == gridDim.x - 1;
    }
  }
  if (!DOTS) return;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double s0 = 0.0, s1 = 0.0;                                    // row order, fixed shape
  for (int q = tid; q < (int)gridDim.x; q += NT) { s0 += __ldcg(a.lrowd + 2 * q); s1 += __ldcg(a.lrowd + 2 * q + 1); }
  block_sum2(s0, s1, sm);
  __shared__ int s_fin;
  if (tid == 0) {
    *a.lcounter = 0u;
    a.partial[0] = s0;
    a.partial[1] = s1;
    s_fin = 0;
    if (a.finalize) {                                 // one more arrival in the slices' election
      __threadfence();
      s_fin = atomicAdd(a.counter, 1u) == (unsigned)(a.elect_total - 1);
    }
  }
  __syncthreads();
  if (!s_fin) return;
  __threadfence();
  if (tid == 0) *a.counter = 0u;
  double t0 = 0.0, t1 = 0.0;
  final_sum2(a.part_base, a.nparts, t0, t1, sm);
  if (tid != 0) return;
  if (ROLE == ROLE_K1) {
    if (a.dist) *a.rho_out = t0;
    else tail_rho(a.ctl, a.rec, t0);
  } else if (ROLE == ROLE_K2DOTS) {
    tail_y(a.ctl, a.rec, t0, t1);
  }
}

template <int ROLE>
__global__ void __launch_bounds__(NT) k_longchunks(SpmvSeg a) {
  if (a.ctl != nullptr && a.ctl->done) return;
  const bool wtd = ROLE == ROLE_K2DOTS && a.wi != nullptr && a.ctl != nullptr && a.ctl->weighted;
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (NT / 32) + (threadIdx.x >> 5);
  if (c >= a.nchunks) return;
  if (!longchunk_warp<ROLE, LCU>(a, c, a.partial, wtd, lane)) return;
  __threadfence();
  double t0, t1;
  final_sum2_warp(a.part_base, a.nparts, t0, t1);
  if (lane != 0) return;
  *a.counter = 0u;
  if (ROLE == ROLE_K1) {
    if (a.dist) *a.rho_out = t0;
    else tail_rho(a.ctl, a.rec, t0);
  } else if (ROLE == ROLE_K2DOTS) {
    tail_y(a.ctl, a.rec, t0, t1);
  }
}

// K1 / K2 / plain SpMV over SELL-32 with a sliding shared-memory WINDOW of the gathered vector.
// Banded matrices (C3's stencil, C5's band half) gather most entries of a run of rows from a
// narrow range of g. Each CTA walks a contiguous, entry-balanced range of blocks (nsb slices
// each); block b's window g[lo_b, lo_b + win) lives in a ring of `ring` doubles
// (slot = (row + goff) mod ring, goff = 16-byte phase of g), loaded by TMA bulk copies: only the
// rows new to block b, up to WST-1 blocks ahead, one copy landing before the next is issued (a
// block also reads rows earlier copies brought in). Setup keeps lo_b nondecreasing with
// lo_b - lo_{b-WST+1} <= ring - win - 2 so a load never overwrites rows a block still in flight
// may read; otherwise the block is a `reset` (whole window reloaded once all earlier blocks are
// done). Entries inside the window read the ring, the rest gather from global memory. The sum
// order is unchanged (ascending, __dadd_rn/__dmul_rn): bitwise the k_sell result.
// Warp specialization: NWC consumer warps take slices in order from a shared counter (slices of a
// sigma window are longest-first: LPT scheduling), grabbing the next slice and prefetching its
// metadata while the current one runs; one producer warp issues the window loads; full/empty
// mbarriers per stage. Dot partials are reduced per slice and summed in slice order
// (deterministic although slices are taken in a run-dependent order).
// ---------------------------------------------------------------------------------------------
#ifndef PLSS_NWC
#define PLSS_NWC 31
#endif
constexpr int NWC = PLSS_NWC;             // consumer warps per windowed CTA
constexpr int NTW = (NWC + 1) * 32;       // + 1 producer warp
#ifndef PLSS_SUW
#define PLSS_SUW 6
#endif
constexpr int SUW = PLSS_SUW;             // steps in flight per lane (windowed kernel)
#ifndef PLSS_WST
#define PLSS_WST 4
#endif
#ifndef PLSS_WCHECK
#define PLSS_WCHECK 0                     // debug: compare every ring read with global memory
#endif
constexpr int WST = PLSS_WST;             // window pipeline stages (blocks in flight)
__device__ __forceinline__ void mbar_arrive_cnt(uint64_t* bar, unsigned cnt) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(cnt) : "memory");
}

template <int ROLE>
__global__ void __launch_bounds__(NTW, 1) k_sellw(SpmvSeg a) {
  extern __shared__ __align__(128) double ring[];
  __shared__ uint64_t full[WST], empty[WST];
  __shared__ int s_next;
  __shared__ volatile int s_issued;                // last block (relative) whose load was issued
  __shared__ double sm[2][MAXW];
  if (a.ctl != nullptr && a.ctl->done) return;
  const bool wtd = ROLE == ROLE_K2DOTS && a.wi != nullptr && a.ctl != nullptr && a.ctl->weighted;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nsb = a.nsb;
  const int b0 = a.cblk[blockIdx.x], b1 = a.cblk[blockIdx.x + 1];
  const int sl0 = b0 * nsb, sl1 = min(b1 * nsb, a.nslices);
  const int W = a.win, R = a.ring;
  const int goff = (int)((reinterpret_cast<uintptr_t>(a.g) >> 3) & 1);
  // window start of block b with the 16-byte phase of this g (setup used the phase of its g)
  auto lo_of = [&](int lo) {
    if ((lo + goff) & 1) lo += lo > 0 ? -1 : 1;
    return lo;
  };
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < WST; ++q) { mbar_init(&full[q], 1); mbar_init(&empty[q], (unsigned)nsb); }
    s_next = sl0 + NWC;                              // slices sl0 .. sl0+NWC-1 are taken statically
    s_issued = -1;
    fence_mbar_init();
  }
  __syncthreads();
  double acc0 = 0.0, acc1 = 0.0;

  if (warp == NWC) {
    // ---- producer: window loads -------------------------------------------------------------
    if (lane == 0) {
      const uint64_t pol_g = a.pol_last;
      int cur = -1;                                  // lo of the window in the ring (-1: none)
      int waited = -1;                               // blocks <= waited (relative) are done
      auto wait_done = [&](int jj) {                 // wait until relative blocks <= jj are done
        for (int k = waited + 1; k <= jj; ++k) mbar_wait(&empty[k % WST], (unsigned)(k / WST) & 1u);
        if (jj > waited) waited = jj;
      };
      for (int b = b0; b < b1; ++b) {
        const int j = b - b0, q = j % WST;
        const int2 wb = a.wlo[b];
        wait_done(j - WST);                          // stage q is free
        const bool nowin = wb.y & 2;
        const bool reset = !nowin && (cur < 0 || (wb.y & 1));
        if (reset) wait_done(j - 1);                 // nothing in flight reads the ring
        const int lo = lo_of(wb.x);
        const int from = nowin ? 0 : reset ? lo : max(lo, cur + W), to = nowin ? 0 : lo + W;
        if (!nowin) cur = lo;
        unsigned bytes = 0;
        fence_proxy_async();
        if (to > from) {
          const int s = (from + goff) % R;
          const int n1 = min(to - from, R - s);
          tma_load(ring + s, a.g + from, (unsigned)n1 * 8u, &full[q], pol_g);
          bytes = (unsigned)n1 * 8u;
          if (to - from > n1) {
            tma_load(ring, a.g + from + n1, (unsigned)(to - from - n1) * 8u, &full[q], pol_g);
            bytes += (unsigned)(to - from - n1) * 8u;
          }
        }
        mbar_expect_tx(&full[q], bytes);
#if PLSS_WCHECK
        if (blockIdx.x < 4) printf("WLOAD cta %d b %d j %d lo %d flags %d reset %d from %d to %d cur %d\n", blockIdx.x, b, j, lo, wb.y, (int)reset, from, to, cur);
#endif
        const int cnt = min((b + 1) * nsb, a.nslices) - b * nsb;     // partial last block
        if (cnt < nsb) mbar_arrive_cnt(&empty[q], (unsigned)(nsb - cnt));
        // Loads land in order: block j reads ring rows that earlier blocks' copies brought in, so
        // "block j's bytes arrived" must imply every earlier copy arrived too.
        mbar_wait(&full[q], (unsigned)(j / WST) & 1u);
        s_issued = j;
      }
    }
    __syncwarp();
  } else {
    // ---- consumers: one slice at a time, in order; the next one's metadata in flight ----------
    const uint64_t pol = a.pol_first;
    int sl = sl0 + warp;                             // first slice: static
    int m0 = 0, m1 = 0, mrow = -1;
    int2 mw = make_int2(0, 0);
    auto meta = [&](int t) {
      m0 = a.sptr[t]; m1 = a.sptr[t + 1];
      mrow = a.perm ? a.perm[t * 32 + lane] : t * 32 + lane;
      mw = a.wlo[t / nsb];
    };
    if (sl < sl1) meta(sl);
    while (sl < sl1) {
      const int st0 = m0, L = m1 - m0, row = mrow;
      const int2 wb = mw;
      int nx = 0;
      if (lane == 0) nx = atomicAdd(&s_next, 1);
      nx = __shfl_sync(FULL, nx, 0);
      if (nx < sl1) meta(nx);
      const int b = sl / nsb, j = b - b0, q = j % WST;
      const int lo = lo_of(wb.x);
      const int Wb = (wb.y & 2) ? 0 : W;             // no window for this block
      const int slo = (lo + goff) % R;
      const bool valid = row >= 0 && row < a.nrows;
      double s = 0.0;
      if (ROLE >= ROLE_K2 && valid && a.accumulate) s = a.out[row];
      const double r_old = (ROLE == ROLE_K1 && valid) ? a.out[row] : 0.0;   // issued early
      const int32_t* ip = a.idx + (long long)st0 * 32 + lane;
      const double* vp = a.val + (long long)st0 * 32 + lane;
      // Parity waits alias across two phases: wait on block j's phase only once j was issued
      // (issuing j required block j-WST done, so stage q's barrier is exactly at j's phase).
      if (s_issued < j) {
        const long long t0 = clock64();
        while (s_issued < j) { __nanosleep(64); spin_guard(t0); }
      }
      mbar_wait(&full[q], (unsigned)(j / WST) & 1u);
      auto gather = [&](int c) -> double {
        const unsigned d = (unsigned)(c - lo);
        if (d < (unsigned)Wb) {
          int k = slo + (int)d;
          if (k >= R) k -= R;
#if PLSS_WCHECK
          const double rv = ring[k], gvv = __ldg(a.g + c);
          if (__double_as_longlong(rv) != __double_as_longlong(gvv))
            printf("WCHECK blk %d cta %d b %d j %d sl %d c %d lo %d W %d R %d slo %d k %d flags %d issued %d\n",
                   blockIdx.x, blockIdx.x, b, j, sl, c, lo, W, R, slo, k, wb.y, (int)s_issued);
          return rv;
#else
          return ring[k];
#endif
        }
        return c >= 0 ? __ldg(a.g + c) : 0.0;
      };
      int jj = 0;
      for (; jj + SUW <= L; jj += SUW) {
        int32_t c[SUW];
        double v[SUW], gv[SUW];
#pragma unroll
        for (int u = 0; u < SUW; ++u) { c[u] = ld_stream(ip + (jj + u) * 32, pol); v[u] = ld_stream(vp + (jj + u) * 32, pol); }
#pragma unroll
        for (int u = 0; u < SUW; ++u) gv[u] = gather(c[u]);
#pragma unroll
        for (int u = 0; u < SUW; ++u) if (c[u] >= 0) s = __dadd_rn(s, __dmul_rn(v[u], gv[u]));
      }
      if (jj < L) {
        int32_t c[SUW];
        double v[SUW], gv[SUW];
#pragma unroll
        for (int u = 0; u < SUW; ++u) {
          c[u] = -1;
          if (jj + u < L) { c[u] = ld_stream(ip + (jj + u) * 32, pol); v[u] = ld_stream(vp + (jj + u) * 32, pol); }
        }
#pragma unroll
        for (int u = 0; u < SUW; ++u) gv[u] = gather(c[u]);
#pragma unroll
        for (int u = 0; u < SUW; ++u) if (c[u] >= 0) s = __dadd_rn(s, __dmul_rn(v[u], gv[u]));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[q]);                    // this slice no longer reads the ring
      double d0 = 0.0, d1 = 0.0;
      if (valid) {
        if (ROLE == ROLE_PLAIN) {
          a.out[row] = s;
        } else if (ROLE == ROLE_K1) {
          const double rn = __dsub_rn(r_old, s);                // r_i <- r_i - (A p)_i
          a.out[row] = rn;
          d0 = rn * rn;
        } else if (ROLE == ROLE_K2DOTS) {
          a.out[row] = k2_final(a, wtd, row, s, d0, d1);   // y_j (WIy_j under PLSS W)
        } else {
          a.out[row] = s;                                       // y_j
        }
      }
      if (ROLE == ROLE_K1 || ROLE == ROLE_K2DOTS) {
        d0 = warp_sum(d0);
        d1 = warp_sum(d1);
        if (lane == 0) { a.slpart[2 * sl] = d0; a.slpart[2 * sl + 1] = d1; }
      }
      sl = nx;
    }
  }
  if (ROLE == ROLE_PLAIN || ROLE == ROLE_K2) return;
  __syncthreads();
  for (int q = sl0 + tid; q < sl1; q += NTW) { acc0 += a.slpart[2 * q]; acc1 += a.slpart[2 * q + 1]; }
  if (!a.finalize) {
    block_sum2(acc0, acc1, sm);
    if (tid == 0) { a.partial[2 * blockIdx.x] = acc0; a.partial[2 * blockIdx.x + 1] = acc1; }
    return;
  }
  if (!publish_and_elect(acc0, acc1, a.partial, a.part_base, a.nparts, a.counter, sm)) return;
  if (tid != 0) return;
  if (ROLE == ROLE_K1) {
    if (a.dist) *a.rho_out = acc0;
    else tail_rho(a.ctl, a.rec, acc0);
  } else if (ROLE == ROLE_K2DOTS) {
    tail_y(a.ctl, a.rec, acc0, acc1);
  }
}

// ---- window choice (setup, once per segment) ------------------------------------------------
// Block b: histogram of its gathered indices in bins of bw; the window starts where `kb`
// consecutive bins hold the most entries (ties: lowest); then clamped to [0, glen - win - 2] and
// given the 16-byte phase of g. A block whose window would hold fewer than `thr` entries gets no
// window (flag 2: loading it would cost more than it saves); the others add their exact
// in-window count to *covered.
__global__ void __launch_bounds__(256) k_win_choose(const int32_t* sptr, const int32_t* sidx, int nslices,
                                                    int nsb, int glen, int win, int bw, int nbins, int kb, int goff,
                                                    int thr, int2* wlo, unsigned long long* covered) {
  extern __shared__ int32_t hist[];
  __shared__ int s_cnt[8], s_pos[8];
  __shared__ unsigned s_sum[8];
  const int b = blockIdx.x, t = threadIdx.x;
  const long long e0 = (long long)sptr[b * nsb] * 32, e1 = (long long)sptr[min((b + 1) * nsb, nslices)] * 32;
  for (int i = t; i < nbins; i += 256) hist[i] = 0;
  __syncthreads();
  for (long long e = e0 + t; e < e1; e += 256) {
    const int c = sidx[e];
    if (c >= 0) atomicAdd(&hist[c / bw], 1);
  }
  __syncthreads();
  int best = -1, bpos = 0;
  const int ncand = max(1, nbins - kb + 1);
  for (int i = t; i < ncand; i += 256) {
    int sum = 0;
    for (int q = 0; q < kb && i + q < nbins; ++q) sum += hist[i + q];
    if (sum > best) { best = sum; bpos = i; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const int ob = __shfl_xor_sync(FULL, best, o), op = __shfl_xor_sync(FULL, bpos, o);
    if (ob > best || (ob == best && op < bpos)) { best = ob; bpos = op; }
  }
  if ((t & 31) == 0) { s_cnt[t >> 5] = best; s_pos[t >> 5] = bpos; }
  __syncthreads();
  __shared__ int s_lo;
  if (t == 0) {
    for (int w = 1; w < 8; ++w)
      if (s_cnt[w] > best || (s_cnt[w] == best && s_pos[w] < bpos)) { best = s_cnt[w]; bpos = s_pos[w]; }
    long long lo = (long long)bpos * bw - (long long)(win - kb * bw) / 2;
    lo = max(0ll, min(lo, (long long)glen - win - 2));
    if ((lo + goff) & 1) lo += lo > 0 ? -1 : 1;
    s_lo = (int)lo;
  }
  __syncthreads();
  const int lo = s_lo;
  unsigned cnt = 0;
  for (long long e = e0 + t; e < e1; e += 256) cnt += (unsigned)(sidx[e] - lo) < (unsigned)win;
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
  if ((t & 31) == 0) s_sum[t >> 5] = cnt;
  __syncthreads();
  if (t == 0) {
    unsigned tot = 0;
    for (int w = 0; w < 8; ++w) tot += s_sum[w];
    const bool use = (int)tot >= thr;
    wlo[b] = make_int2(lo, use ? 0 : 2);
    if (use) atomicAdd(covered, (unsigned long long)tot);
  }
}

// Per CTA range (the grid is fixed at setup): keep the windows of the windowed blocks
// nondecreasing with lo_b - lo_k <= ring - win - 2 for every windowed block k among the WST-1
// blocks before b (those may still be in flight while b's rows are loaded). Small violations are
// clamped, large ones become `reset` blocks (flag 1). Blocks without a window (flag 2) are
// transparent.
__global__ void k_win_chain(int2* wlo, const int32_t* cblk, int grid, int win, int ring) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= grid) return;
  const int b0 = cblk[c], b1 = cblk[c + 1];
  const int adv = ring - win - 2, slack = win / 8;
  int prev = -1;                                 // lo of the last windowed block
  int hist[WST];                                 // lo of the last WST-1 blocks (-1: no window)
  for (int k = 0; k < WST; ++k) hist[k] = -1;
  for (int b = b0; b < b1; ++b) {
    int2 w = wlo[b];
    const int slot = (b - b0) % WST;
    if (w.y & 2) { hist[slot] = -1; continue; }
    int oldest = -1;                             // smallest lo among the in-flight window blocks
    for (int k = 1; k < WST; ++k) {
      const int h = hist[((b - b0) - k + WST * 4) % WST];
      if ((b - b0) - k >= 0 && h >= 0 && (oldest < 0 || h < oldest)) oldest = h;
    }
    int lo = w.x, reset = 0;
    if (prev < 0) {
      reset = 1;
    } else if (lo < prev) {
      if (prev - lo <= slack) lo = prev; else reset = 1;
    }
    if (!reset && oldest >= 0 && lo - oldest > adv) {
      if (lo - oldest - adv <= slack) lo = oldest + adv; else reset = 1;
      if (!reset && lo < prev) lo = prev;        // cannot happen with monotone windows; keep safe
      if (!reset && lo - oldest > adv) reset = 1;
    }
    wlo[b] = make_int2(lo, reset);
    hist[slot] = lo;
    prev = lo;
  }
}

// CTA c of a windowed launch owns blocks [cblk[c], cblk[c+1]): the first block whose stored
// entries start at or after c/grid of the segment's total (work balance when row lengths vary,
// e.g. C5's K2 slabs where a band of columns holds 9x the entries of the rest).
// out = {sum (b - ax)^2, sum b^2} over this rank's rows: fixed per-thread order, block trees, last
// CTA sums the CTA pairs in index order (deterministic). plss_true_residual.
__global__ void __launch_bounds__(NT) k_true_resid(const double* __restrict__ b, const double* __restrict__ ax,
                                                   long long m, double* part, unsigned* counter, double* out) {
  __shared__ double sm[2][MAXW];
  double s0 = 0.0, s1 = 0.0;
  for (long long i = (long long)blockIdx.x * NT + threadIdx.x; i < m; i += (long long)gridDim.x * NT) {
    const double d = __dadd_rn(b[i], -ax[i]);
    s0 = __dadd_rn(s0, __dmul_rn(d, d));
    s1 = __dadd_rn(s1, __dmul_rn(b[i], b[i]));
  }
  if (!publish_and_elect(s0, s1, part, part, gridDim.x, counter, sm)) return;
  if (threadIdx.x == 0) { out[0] = s0; out[1] = s1; }
}

// *out = max_i (row_ptr[i+1] - row_ptr[i]) over i < m (atomicMax; order-independent)
__global__ void k_max_row_len(const int32_t* __restrict__ row_ptr, long long m, int32_t* out) {
  int32_t mx = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
    mx = max(mx, row_ptr[i + 1] - row_ptr[i]);
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx > 0) atomicMax(out, mx);
}

__global__ void k_cta_ranges(const int32_t* w, int wscale, int nunits, int nsb, int nblocks, int grid,
                             int32_t* cblk, int unit_cost, int s1beg = 0x7fffffff, int s1_cost = 0) {
  // w: prefix over units (nunits+1 entries); unit cost = (w[u+1] - w[u]) * wscale + UNIT_COST
  // (a unit also costs its metadata loads, row outputs and dot partial: without that term the
  // empty slices of a segment -- C4's empty columns sort last -- all fall to the last CTA);
  // units from s1beg on (k_sell's batched one-step slices) cost s1_cost instead of UNIT_COST
  const long long UNIT_COST = unit_cost;
  auto pre = [&](int u) -> long long {
    return (long long)w[u] * wscale + (long long)u * UNIT_COST -
           (long long)max(0, u - s1beg) * (UNIT_COST - s1_cost);
  };
  const long long total = pre(nunits);
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c <= grid; c += gridDim.x * blockDim.x) {
    const long long target = (total * c + grid - 1) / grid;
    int lo = 0, hi = nblocks;                                   // first b with start(b) >= target
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      const int u = min(mid * nsb, nunits);
      if (pre(u) < target) lo = mid + 1; else hi = mid;
    }
    cblk[c] = c == 0 ? 0 : c == grid ? nblocks : lo;
  }
}

// ---- SELL-32 construction (setup, once per segment) ------------------------------------------
__global__ void k_max_len(const int32_t* ptr, long long nrows, int* mx) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int l = i < nrows ? ptr[i + 1] - ptr[i] : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) l = max(l, __shfl_xor_sync(FULL, l, o));
  if ((threadIdx.x & 31) == 0 && l > 0) atomicMax(mx, l);
}
__global__ void k_row_len(const int32_t* ptr, long long nrows, int32_t* len) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nrows) len[i] = ptr[i + 1] - ptr[i];
}
// sigma-sort: within each window of SIGMA rows, slots ordered by length descending (stable)
constexpr int SIGMA_NT = SIGMA < 256 ? SIGMA : 256;   // threads of the sigma-sort kernel
template <int SIGMA = plss::SIGMA>
__global__ void __launch_bounds__(SIGMA_NT) k_sigma_sort(const int32_t* len, long long nrows, long long nslots,
                                                         int32_t* perm) {
  // stable radix sort of the window by (length descending, row ascending); missing rows last
  constexpr int IPT = SIGMA / SIGMA_NT;
  using Sort = cub::BlockRadixSort<unsigned, SIGMA_NT, IPT, int32_t>;
  __shared__ typename Sort::TempStorage tmp;
  const long long w0 = (long long)blockIdx.x * SIGMA;
  unsigned key[IPT];
  int32_t val[IPT];
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const long long i = w0 + (long long)threadIdx.x * IPT + k;     // blocked arrangement
    key[k] = i < nrows ? 0x7fffffffu - (unsigned)len[i] : 0xffffffffu;
    val[k] = i < nrows ? (int32_t)i : -1;
  }
  Sort(tmp).Sort(key, val);
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const long long o = w0 + (long long)threadIdx.x * IPT + k;
    if (o < nslots) perm[o] = val[k];
  }
}
__global__ void k_slice_len(const int32_t* len, const int32_t* perm, long long nrows, long long nslices,
                            int32_t* slen) {
  const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (s > nslices) return;
  if (s == nslices) { slen[s] = 0; return; }
  int mx = 0;
  for (int l = 0; l < 32; ++l) {
    const long long slot = s * 32 + l;
    const long long row = perm ? perm[slot] : slot;
    if (row >= 0 && row < nrows) mx = max(mx, len[row]);
  }
  slen[s] = mx;
}
// thread per slot: copy its row's entries (column-major within the slice), pad with index -1
__global__ void k_sell_fill(const int32_t* ptr, const int32_t* idx, const double* val, const int32_t* perm,
                            long long nrows, long long nslices, const int32_t* sptr, int32_t* sidx,
                            double* sval) {
  const long long slot = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= nslices * 32) return;
  const long long s = slot >> 5;
  const int lane = (int)(slot & 31);
  const long long row = perm ? perm[slot] : slot;
  const int L = sptr[s + 1] - sptr[s];
  long long b = 0, e = 0;
  if (row >= 0 && row < nrows) { b = ptr[row]; e = ptr[row + 1]; }
  for (int j = 0; j < L; ++j) {
    const long long dst = ((long long)sptr[s] + j) * 32 + lane;
    if (b + j < e) { sidx[dst] = idx[b + j]; sval[dst] = val[b + j]; }
    else { sidx[dst] = -1; sval[dst] = 0.0; }
  }
}

// ---------------------------------------------------------------------------------------------
// K3: p <- beta p + gamma y; theta = p^T p; x <- x + p  (L811-813); init: p = gamma y (L795)
// ---------------------------------------------------------------------------------------------
constexpr int K3_PSI = 1, K3_XDEFER = 2;         // k_pxupdate options (one device, PLSS path)
#ifndef PLSS_K3X
#define PLSS_K3X 1                                   // K3 loads x together with y and p
#endif
#ifndef PLSS_K3U
#define PLSS_K3U 1                                   // K3 loop unroll
#endif
constexpr int K3U = PLSS_K3U;

// plss_finish under K3_XDEFER: x <- x + p when x lags (Ctl::xlag; the host clears the flag after)
__global__ void __launch_bounds__(NT, VEC_MINB) k_xflush(double* __restrict__ x, const double* __restrict__ p,
                                                       long long n, const Ctl* c) {
  if (!c->xlag) return;
  for (long long i = (long long)blockIdx.x * NT + threadIdx.x; i < n; i += (long long)gridDim.x * NT)
    x[i] = __dadd_rn(x[i], p[i]);
}

// theta_out != NULL (the reduce-scatter distributed step, K3 on this rank's column shard): the
// shard's p^T p goes there (summed across ranks with the next step's scalars) instead of c->theta
__global__ void __launch_bounds__(NT, VEC_MINB) k_pxupdate(double* __restrict__ p, const double* __restrict__ y,
                                                 double* __restrict__ x, long long n, Ctl* c,
                                                 double* rec, double* partial, unsigned* counter,
                                                 const double* __restrict__ wi, double* theta_out = nullptr,
                                                 int opts = 0) {
  __shared__ double sm[2][MAXW];
  if (c->done) return;
  const bool wtd = wi != nullptr && c->weighted;       // theta = p^T (WI p) under PLSS W (L812)
  const int k = c->iters;
  const bool init = (k == 0);
  const double beta = c->beta, gamma = c->gamma;
  // psi = y_k^T p_{k-1} (L806, diagnostic) summed here when K2 left it (SpmvSeg::psi3, WI = I)
  const bool psi = (opts & K3_PSI) && !wtd && !init;
  // K3_XDEFER: x is updated every other step, x <- (x + p_{k-1}) + p_k when it lags (bitwise the
  // two sequential updates of L813); the other steps leave x (Ctl::xlag, plss_finish applies it)
  const bool defer = opts & K3_XDEFER;
  const bool lag = defer && c->xlag;
  double acc = 0.0, acc1 = 0.0;
  const long long n2 = n >> 1;
  const long long stride = (long long)gridDim.x * NT;
  double2* p2 = reinterpret_cast<double2*>(p);
  double2* x2 = reinterpret_cast<double2*>(x);
  const double2* y2 = reinterpret_cast<const double2*>(y);
  const bool xupd = !defer || lag;
#pragma unroll K3U
  for (long long i = (long long)blockIdx.x * NT + threadIdx.x; i < n2; i += stride) {
    const double2 yy = __ldcs(y2 + i);
    double2 pp, po = make_double2(0.0, 0.0);
#if PLSS_K3X
    double2 xx = make_double2(0.0, 0.0);
    if (xupd) xx = __ldcs(x2 + i);                   // issued with y and p: one latency per element
#endif
    if (init) {
      pp.x = __dmul_rn(gamma, yy.x);
      pp.y = __dmul_rn(gamma, yy.y);
    } else {
      po = p2[i];
      pp.x = __dadd_rn(__dmul_rn(beta, po.x), __dmul_rn(gamma, yy.x));
      pp.y = __dadd_rn(__dmul_rn(beta, po.y), __dmul_rn(gamma, yy.y));
      if (psi) {
        acc1 = fma(yy.x, po.x, acc1);
        acc1 = fma(yy.y, po.y, acc1);
      }
    }
    p2[i] = pp;
    if (xupd) {
#if !PLSS_K3X
      double2 xx = __ldcs(x2 + i);
#endif
      if (lag) {
        xx.x = __dadd_rn(xx.x, po.x);
        xx.y = __dadd_rn(xx.y, po.y);
      }
      xx.x = __dadd_rn(xx.x, pp.x);
      xx.y = __dadd_rn(xx.y, pp.y);
      __stcs(x2 + i, xx);
    }
    if (wtd) {
      const double2 w = __ldg(reinterpret_cast<const double2*>(wi) + i);
      acc = fma(pp.x, w.x * pp.x, acc);
      acc = fma(pp.y, w.y * pp.y, acc);
    } else {
      acc = fma(pp.x, pp.x, acc);
      acc = fma(pp.y, pp.y, acc);
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const long long i = n - 1;
    if (psi) acc1 = fma(y[i], p[i], acc1);
    const double po = init ? 0.0 : p[i];
    const double pp = init ? __dmul_rn(gamma, y[i]) : __dadd_rn(__dmul_rn(beta, po), __dmul_rn(gamma, y[i]));
    p[i] = pp;
    if (!defer || lag) x[i] = __dadd_rn(lag ? __dadd_rn(x[i], po) : x[i], pp);
    acc = fma(pp, wtd ? wi[i] * pp : pp, acc);
  }
  if (!publish_and_elect(acc, acc1, partial, partial, gridDim.x, counter, sm)) return;
  if (threadIdx.x != 0) return;
  if (psi) {
    c->psi = acc1;
    rec[(size_t)k * REC + 3] = acc1;
  }
  if (defer) c->xlag = lag ? 0 : 1;
  if (theta_out) {
    *theta_out = acc;                                           // shard partial of theta
  } else {
    c->theta = acc;                                             // theta = p^T p (L812)
    rec[(size_t)k * REC + 4] = acc;
  }
  c->iters = k + 1;
  if (k + 1 >= c->maxit) {
    c->done = 1;
    if (!c->stopped) c->outcome = OUT_MAXIT;
  }
}

// ---------------------------------------------------------------------------------------------
// distributed: phi, psi over the replicated (all-reduced) y, then both tails (K2b)
// ---------------------------------------------------------------------------------------------
// reduce-scatter distributed step: partials of phi = y^T (WI y) and psi = y^T p over this rank's
// column shard (y <- WIy in place under PLSS W), into scal[1], scal[2] (scal[0] = the local rho
// from K1, scal[3] = the shard's theta from the previous K3); then one all-reduce of scal[0..3]
__global__ void __launch_bounds__(NT) k_dots_shard(double* __restrict__ y, const double* __restrict__ p,
                                                   long long nsh, Ctl* c, double* partial, unsigned* counter,
                                                   const double* __restrict__ wi, double* scal) {
  __shared__ double sm[2][MAXW];
  if (c->done) return;
  const bool wtd = wi != nullptr && c->weighted;
  double a0 = 0.0, a1 = 0.0;
  for (long long i = (long long)blockIdx.x * NT + threadIdx.x; i < nsh; i += (long long)gridDim.x * NT) {
    const double yy = y[i];
    if (wtd) {
      const double wy = __ddiv_rn(yy, wi[i]);
      y[i] = wy;
      a0 = fma(yy, wy, a0);
      a1 = fma(wy, p[i], a1);
    } else {
      a0 = fma(yy, yy, a0);
      a1 = fma(yy, p[i], a1);
    }
  }
  if (!publish_and_elect(a0, a1, partial, partial, gridDim.x, counter, sm)) return;
  if (threadIdx.x == 0) { scal[1] = a0; scal[2] = a1; }
}

// the replicated scalar tails from the all-reduced scal = {rho, phi, psi, theta of p_{k-1}}
__global__ void k_tail_rsag(Ctl* c, double* rec, const double* scal) {
  if (c->done) return;
  const int k = c->iters;
  if (k > 0) {
    c->theta = scal[3];
    rec[(size_t)(k - 1) * REC + 4] = scal[3];
  }
  tail_rho(c, rec, scal[0]);
  if (!c->done) tail_y(c, rec, scal[1], scal[2]);
}

// column-block distributed step (plss_create_dist_cols, SURVEY 8(e) "column-block alternative"):
// r is replicated and was just all-reduced (r <- r - sum_g A_g p_g, with r[m] = sum_g theta_g of the
// previous K3); rho = r^T r (every rank the same fixed-order sum of the same bytes), theta, the
// stop test and the rho tail
__global__ void __launch_bounds__(NT, VEC_MINB) k_rho_tail(const double* __restrict__ r, long long m, Ctl* c,
                                                 double* rec, double* partial, unsigned* counter) {
  __shared__ double sm[2][MAXW];
  if (c->done) return;
  double a0 = 0.0, dummy = 0.0;
  for (long long i = (long long)blockIdx.x * NT + threadIdx.x; i < m; i += (long long)gridDim.x * NT)
    a0 = fma(r[i], r[i], a0);
  if (!publish_and_elect(a0, dummy, partial, partial, gridDim.x, counter, sm)) return;
  if (threadIdx.x != 0) return;
  const int k = c->iters;
  if (k > 0) {
    c->theta = r[m];
    rec[(size_t)(k - 1) * REC + 4] = r[m];
  }
  tail_rho(c, rec, a0);
}

// column-block step: the y tail from the all-reduced scal[1] = phi, scal[2] = psi
__global__ void k_tail_phi(Ctl* c, double* rec, const double* scal) {
  if (c->done) return;
  tail_y(c, rec, scal[1], scal[2]);
}

__global__ void __launch_bounds__(NT) k_dots_tail(double* __restrict__ y, const double* __restrict__ p,
                                                  long long n, const double* rho_g, Ctl* c,
                                                  double* rec, double* partial, unsigned* counter,
                                                  const double* __restrict__ wi, int psi_k3 = 0) {
  __shared__ double sm[2][MAXW];
  if (c->done) return;
  const bool wtd = wi != nullptr && c->weighted;
  const bool psi = !psi_k3 || wtd;                 // else K3 sums psi (K3_PSI) and p is not read here
  double a0 = 0.0, a1 = 0.0;
  auto one = [&](long long i) {
    const double yy = y[i];
    if (wtd) {                                      // y <- WIy in place (what K3 consumes)
      const double wy = __ddiv_rn(yy, wi[i]);
      y[i] = wy;
      a0 = fma(yy, wy, a0);
    } else {
      a0 = fma(yy, yy, a0);
    }
    if (psi) a1 = fma(yy, p[i], a1);
  };
  const long long stride = (long long)gridDim.x * NT;
  if (((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(wi)) & 15) == 0) {
    // 16-byte loads of element pairs; the odd last element by thread 0 of CTA 0
    const long long n2 = n >> 1;
    for (long long i = (long long)blockIdx.x * NT + threadIdx.x; i < n2; i += stride) {
      const double2 yy = reinterpret_cast<const double2*>(y)[i];
      const double2 pp = psi ? reinterpret_cast<const double2*>(p)[i] : make_double2(0.0, 0.0);
      if (wtd) {
        const double2 ww = reinterpret_cast<const double2*>(wi)[i];
        const double2 wy = make_double2(__ddiv_rn(yy.x, ww.x), __ddiv_rn(yy.y, ww.y));
        reinterpret_cast<double2*>(y)[i] = wy;
        a0 = fma(yy.x, wy.x, a0);
        a0 = fma(yy.y, wy.y, a0);
      } else {
        a0 = fma(yy.x, yy.x, a0);
        a0 = fma(yy.y, yy.y, a0);
      }
      a1 = fma(yy.x, pp.x, a1);
      a1 = fma(yy.y, pp.y, a1);
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) one(n - 1);
  } else {
    for (long long i = (long long)blockIdx.x * NT + threadIdx.x; i < n; i += stride) one(i);
  }
  if (!publish_and_elect(a0, a1, partial, partial, gridDim.x, counter, sm)) return;
  if (threadIdx.x != 0) return;
  tail_rho(c, rec, *rho_g);
  if (c->done) return;
  tail_y(c, rec, a0, a1);
}

// ||b||^2 (or the local share of it) into ctl->nb2; non-dist also sets nbd.
__global__ void __launch_bounds__(NT, VEC_MINB) k_norm_b(const double* __restrict__ r, long long m, Ctl* c,
                                               double* partial, unsigned* counter, int set_nbd,
                                               double* out) {
  __shared__ double sm[2][MAXW];
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
// column sums of squares (ascending row order) of a CSC; finish: sqrt, zero columns -> 1
__global__ void k_colsq(const int32_t* col_ptr, const double* val_t, long long n, double* c) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double s = 0.0;
  for (long long k = col_ptr[j]; k < col_ptr[j + 1]; ++k) s = __dadd_rn(s, __dmul_rn(val_t[k], val_t[k]));
  c[j] = s;
}
__global__ void k_colnorm_finish(double* c, long long n) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) c[j] = c[j] > 0.0 ? __dsqrt_rn(c[j]) : 1.0;
}
__global__ void k_check_positive(const double* w, long long n, int* err) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n && !(w[j] > 0.0 && isfinite(w[j]))) atomicOr(err, 1);
}
__global__ void k_policies(uint64_t* out) {
  out[0] = policy_evict_first();
  out[1] = policy_evict_last();
}

__device__ __forceinline__ int lower_bound_pos(const int32_t* ptr, int nrows, long long key) {
  int lo = 0, hi = nrows;
  while (lo < hi) {
    const int mid = lo + ((hi - lo) >> 1);
    if ((long long)ptr[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// tile construction (setup): a new tile starts at row i when the TILE-window of its first entry
// or its RCAP-row block differs from row i-1's
__device__ __forceinline__ int tile_flag(const int32_t* ptr, long long i, long long e0) {
  if (i == 0) return 1;
  return ((ptr[i] - e0) / TILE != (ptr[i - 1] - e0) / TILE) || (i / RCAP != (i - 1) / RCAP);
}
__global__ void k_tile_mark(const int32_t* ptr, long long nrows, long long e0, int32_t* flag) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nrows) flag[i] = tile_flag(ptr, i, e0);
  else if (i == nrows) flag[i] = 0;
}
// after the exclusive scan: pos[i] = tile index of row i if it starts a tile
__global__ void k_tile_desc(const int32_t* ptr, long long nrows, long long e0, const int32_t* pos,
                            int2* desc) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nrows) {
    if (tile_flag(ptr, i, e0)) desc[pos[i]] = make_int2((int)i, ptr[i]);
  } else if (i == nrows) {
    desc[pos[nrows]] = make_int2((int)nrows, ptr[nrows]);
  }
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
