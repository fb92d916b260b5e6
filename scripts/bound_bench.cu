// Microbenchmark: what bounds K1 / K2 on C5 ("settle what bounds the kernel
// with a microbenchmark that replays C5's exact band and uniform index streams, with and without
// the value / index streams; explain the band-free ablation").
//
// One C5 slab (6.4M rows of the 64M x 8M matrix, rows of 12 entries: 6 in the band window
// [lo_i, lo_i + 2048], lo_i = clip(i/8 - 1024, 0, n - 2049), 6 uniform; SELL-32 column-major as
// libplss stores it), and the band half of the slab's transpose (the 0.8M columns whose band rows
// lie in the slab, 48 band entries each). Every kernel variant is timed with CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o bound_bench bound_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
#include "../paper_2207_07615_b200/csrc/plss_kernels.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

constexpr long long N = 8000000;          // columns
constexpr long long M = 64000000;         // rows of the whole matrix
constexpr int RS = 6400000;               // rows of one slab
constexpr long long OFF = 3ll * RS;       // the slab's first row (a middle slab)
constexpr int L = 12;                     // entries per row
constexpr int NB = 6;                     // band entries per row

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ long long band_lo(long long gi) {
  long long lo = gi / 8 - 1024;
  return lo < 0 ? 0 : (lo > N - 2049 ? N - 2049 : lo);
}

// K1 slab in SELL-32 (slice s, step j, lane l at (s*L + j)*32 + l); also the split layout: the
// band entries (6 steps) and the uniform entries (6 steps) as two SELL arrays.
__global__ void gen_k1(int32_t* idx, double* val, int32_t* bidx, double* bval, int32_t* uidx, double* uval) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= RS) return;
  const long long gi = OFF + i, lo = band_lo(gi);
  long long c[L];
  uint64_t h = mix(gi * 7919ull);
  for (int k = 0; k < L; ++k) {
    for (;;) {
      h = mix(h);
      const long long cand = k < NB ? lo + (long long)(h % 2049) : (long long)(h % N);
      bool dup = false;
      for (int q = 0; q < k; ++q) dup |= c[q] == cand;
      if (!dup) { c[k] = cand; break; }
    }
  }
  double v[L];
  for (int k = 0; k < L; ++k) { h = mix(h); v[k] = (double)(h % 2000001) * 1e-6 - 1.0; }
  // split layout first (band, uniform, each ascending)
  for (int a = 0; a < NB; ++a) for (int b = a + 1; b < NB; ++b) if (c[b] < c[a]) { long long t = c[a]; c[a] = c[b]; c[b] = t; double tv = v[a]; v[a] = v[b]; v[b] = tv; }
  for (int a = NB; a < L; ++a) for (int b = a + 1; b < L; ++b) if (c[b] < c[a]) { long long t = c[a]; c[a] = c[b]; c[b] = t; double tv = v[a]; v[a] = v[b]; v[b] = tv; }
  const long long s = i / 32, l = i % 32;
  for (int k = 0; k < NB; ++k) {
    bidx[(s * NB + k) * 32 + l] = (int32_t)c[k]; bval[(s * NB + k) * 32 + l] = v[k];
    uidx[(s * (L - NB) + k) * 32 + l] = (int32_t)c[NB + k]; uval[(s * (L - NB) + k) * 32 + l] = v[NB + k];
  }
  for (int a = 0; a < L; ++a) for (int b = a + 1; b < L; ++b) if (c[b] < c[a]) { long long t = c[a]; c[a] = c[b]; c[b] = t; double tv = v[a]; v[a] = v[b]; v[b] = tv; }
  for (int k = 0; k < L; ++k) { idx[(s * L + k) * 32 + l] = (int32_t)c[k]; val[(s * L + k) * 32 + l] = v[k]; }
}

__device__ __forceinline__ double lds_stream(const double* p) {
  double v; asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p)); return v;
}
__device__ __forceinline__ int32_t ldi_stream(const int32_t* p) {
  int32_t v; asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p)); return v;
}

// MODE: 0 full, 1 band gathers skipped (predicated off), 2 uniform gathers skipped, 3 no gathers,
//       4 band gathers from a shared-memory window of p (per chunk of the CTA's slice range),
//       5 no stream loads (indices from the hash, values 1): gathers only
template <int MODE, int BS, int SU>
__global__ void __launch_bounds__(BS, BS == 1024 ? 1 : (BS == 512 ? 2 : 4)) k1(const int32_t* __restrict__ idx, const double* __restrict__ val,
                                                 const double* __restrict__ p, double* __restrict__ r, int nslices,
                                                 int chunk) {
  extern __shared__ double sp[];
  constexpr int NW = BS / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s0 = (int)((long long)nslices * blockIdx.x / gridDim.x), s1 = (int)((long long)nslices * (blockIdx.x + 1) / gridDim.x);
  for (int c0 = s0; c0 < s1; c0 += (MODE == 4 ? chunk : (s1 - s0))) {
    const int c1 = min(s1, c0 + (MODE == 4 ? chunk : (s1 - s0)));
    long long wlo = 0, whi = 0;
    if (MODE == 4) {
      wlo = band_lo(OFF + (long long)c0 * 32);
      whi = band_lo(OFF + (long long)c1 * 32 - 1) + 2049;
      __syncthreads();
      for (long long q = wlo + threadIdx.x; q < whi; q += BS) sp[q - wlo] = __ldg(p + q);
      __syncthreads();
    }
    for (int s = c0 + warp; s < c1; s += NW) {
      const long long row = (long long)s * 32 + lane;
      const long long gi = OFF + row;
      const long long blo = band_lo(gi);
      double sum = 0.0;
      const int32_t* ip = idx + (long long)s * L * 32 + lane;
      const double* vp = val + (long long)s * L * 32 + lane;
      uint64_t h = mix(gi);
#pragma unroll
      for (int j0 = 0; j0 < L; j0 += SU) {
        int32_t c[SU]; double v[SU], g[SU];
#pragma unroll
        for (int u = 0; u < SU; ++u) {
          if (MODE == 5) { h = mix(h); c[u] = (u & 1) ? (int32_t)(blo + h % 2049) : (int32_t)(h % N); v[u] = 1.0; }
          else { c[u] = ldi_stream(ip + (j0 + u) * 32); v[u] = lds_stream(vp + (j0 + u) * 32); }
        }
#pragma unroll
        for (int u = 0; u < SU; ++u) {
          const bool band = c[u] >= blo && c[u] <= blo + 2048;
          if (MODE == 0 || MODE == 5) g[u] = __ldg(p + c[u]);
          else if (MODE == 1) g[u] = band ? 1.0 : __ldg(p + c[u]);
          else if (MODE == 2) g[u] = band ? __ldg(p + c[u]) : 1.0;
          else if (MODE == 3) g[u] = (double)c[u];
          else if (MODE == 4) g[u] = (c[u] >= wlo && c[u] < whi) ? sp[c[u] - wlo] : __ldg(p + c[u]);
          else if (MODE == 6) g[u] = band ? __ldg(p + c[u]) : __ldcg(p + c[u]);
          else if (MODE == 7) { if (band) g[u] = __ldg(p + c[u]); else asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(g[u]) : "l"(p + c[u])); }
          else if (MODE == 8) g[u] = __ldcg(p + c[u]);
          else if (MODE == 9) g[u] = band ? __ldg(p + c[u]) : __ldcs(p + c[u]);
        }
#pragma unroll
        for (int u = 0; u < SU; ++u) sum = __dadd_rn(sum, __dmul_rn(v[u], g[u]));
      }
      r[row] = r[row] - sum;
    }
  }
}


// ---- software-pipelined K1: each warp streams its slices' idx / val steps into its own ring of
// NSTG shared-memory stages (SUB steps each) with cp.async (16-byte LDGSTS, L2 only), NSTG - 1
// stages ahead; the gathers of a stage are issued from shared-memory indices. r_old is loaded at
// the slice's first stage.
__device__ __forceinline__ void cpasync16(void* smem, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"((unsigned)__cvta_generic_to_shared(smem)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N_> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N_) : "memory"); }

template <int SUB, int NSTG, int BS>
__global__ void __launch_bounds__(BS, 2048 / BS / 2) k1p(const int32_t* __restrict__ idx, const double* __restrict__ val,
                                              const double* __restrict__ p, double* __restrict__ r, int nslices) {
  extern __shared__ __align__(16) unsigned char smraw[];
  constexpr int NW = BS / 32, SPS = L / SUB, STB = SUB * 32 * 12;
  static_assert(L % SUB == 0, "SUB divides L");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* ring = smraw + warp * NSTG * STB;
  const int s0 = (int)((long long)nslices * blockIdx.x / gridDim.x), s1 = (int)((long long)nslices * (blockIdx.x + 1) / gridDim.x);
  const int first = s0 + warp;
  const int nsw = first < s1 ? (s1 - first + NW - 1) / NW : 0;
  const int G = nsw * SPS;
  auto issue = [&](int g) {
    if (g < G) {
      const long long sl = first + (long long)(g / SPS) * NW;
      const long long st = sl * L + (g % SPS) * SUB;            // first step of the stage
      unsigned char* dst = ring + (g % NSTG) * STB;
      const unsigned char* gi = reinterpret_cast<const unsigned char*>(idx + st * 32);
      const unsigned char* gv = reinterpret_cast<const unsigned char*>(val + st * 32);
#pragma unroll
      for (int c = lane; c < SUB * 24; c += 32) {
        if (c < SUB * 8) cpasync16(dst + c * 16, gi + c * 16);
        else cpasync16(dst + SUB * 128 + (c - SUB * 8) * 16, gv + (c - SUB * 8) * 16);
      }
    }
    cp_commit();
  };
#pragma unroll
  for (int g = 0; g < NSTG - 1; ++g) issue(g);
  double sum = 0.0, rold = 0.0;
  for (int g = 0; g < G; ++g) {
    issue(g + NSTG - 1);
    const int ch = g % SPS;
    const long long row = (long long)(first + (g / SPS) * NW) * 32 + lane;
    if (ch == 0) rold = r[row];
    cp_wait<NSTG - 1>();
    __syncwarp();
    const unsigned char* src = ring + (g % NSTG) * STB;
    int32_t c[SUB]; double v[SUB], gg[SUB];
#pragma unroll
    for (int u = 0; u < SUB; ++u) {
      c[u] = reinterpret_cast<const int32_t*>(src)[u * 32 + lane];
      v[u] = reinterpret_cast<const double*>(src + SUB * 128)[u * 32 + lane];
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < SUB; ++u) gg[u] = __ldg(p + c[u]);
#pragma unroll
    for (int u = 0; u < SUB; ++u) sum = __dadd_rn(sum, __dmul_rn(v[u], gg[u]));
    if (ch == SPS - 1) { r[row] = rold - sum; sum = 0.0; }
  }
  cp_wait<0>();
}

// the plain kernel with r_old loaded before the row's loads (as libplss does)
template <int SU>
__global__ void __launch_bounds__(1024, 1) k1e(const int32_t* __restrict__ idx, const double* __restrict__ val,
                                              const double* __restrict__ p, double* __restrict__ r, int nslices) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s0 = (int)((long long)nslices * blockIdx.x / gridDim.x), s1 = (int)((long long)nslices * (blockIdx.x + 1) / gridDim.x);
  for (int s = s0 + warp; s < s1; s += 32) {
    const long long row = (long long)s * 32 + lane;
    const double rold = r[row];
    double sum = 0.0;
    const int32_t* ip = idx + (long long)s * L * 32 + lane;
    const double* vp = val + (long long)s * L * 32 + lane;
#pragma unroll
    for (int j0 = 0; j0 < L; j0 += SU) {
      int32_t c[SU]; double v[SU], g[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) { c[u] = ldi_stream(ip + (j0 + u) * 32); v[u] = lds_stream(vp + (j0 + u) * 32); }
#pragma unroll
      for (int u = 0; u < SU; ++u) g[u] = __ldg(p + c[u]);
#pragma unroll
      for (int u = 0; u < SU; ++u) sum = __dadd_rn(sum, __dmul_rn(v[u], g[u]));
    }
    r[row] = rold - sum;
  }
}


// production-like K1 (libplss k_sell<ROLE_K1, 1024>) with each of its per-slice costs switchable:
// F & 1 dynamic slice tickets (shared counter, one slice ahead), F & 2 slice starts loaded from sptr,
// F & 4 per-slice rho partial (warp butterflies of two values + a store), F & 8 L2 evict-first on
// the streams, F & 16 SU 8 + a predicated tail batch (libplss) instead of SU 6 x 2
template <int F>
__global__ void __launch_bounds__(1024, 1) k1x(const int32_t* __restrict__ idx, const double* __restrict__ val,
                                              const double* __restrict__ p, double* __restrict__ r, int nslices,
                                              const int32_t* __restrict__ sptr, double* slpart) {
  __shared__ int s_next;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s0 = (int)((long long)nslices * blockIdx.x / gridDim.x), s1 = (int)((long long)nslices * (blockIdx.x + 1) / gridDim.x);
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (F & 1) { if (threadIdx.x == 0) s_next = s0 + 32; __syncthreads(); }
  int s = s0 + warp;
  int m0 = 0, m1 = 0;
  if ((F & 2) && s < s1) { m0 = sptr[s]; m1 = sptr[s + 1]; }
  double acc = 0.0;
  while (s < s1) {
    int nx;
    if (F & 1) { nx = 0; if (lane == 0) nx = atomicAdd(&s_next, 1); nx = __shfl_sync(0xffffffffu, nx, 0); }
    else nx = s + 32;
    int st0 = s * L, len = L;
    if (F & 2) { st0 = m0; len = m1 - m0; if (nx < s1) { m0 = sptr[nx]; m1 = sptr[nx + 1]; } }
    const long long row = (long long)s * 32 + lane;
    const double rold = r[row];
    double sum = 0.0;
    const int32_t* ip = idx + (long long)st0 * 32 + lane;
    const double* vp = val + (long long)st0 * 32 + lane;
    constexpr int SU = (F & 16) ? 8 : 6;
    for (int j0 = 0; j0 < len; j0 += SU) {
      int32_t c[SU]; double v[SU], g[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        c[u] = -1;
        if (!(F & 16) || j0 + u < len) {
          if (F & 8) {
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(c[u]) : "l"(ip + (j0 + u) * 32), "l"(pol));
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v[u]) : "l"(vp + (j0 + u) * 32), "l"(pol));
          } else { c[u] = ldi_stream(ip + (j0 + u) * 32); v[u] = lds_stream(vp + (j0 + u) * 32); }
        }
      }
#pragma unroll
      for (int u = 0; u < SU; ++u) g[u] = c[u] >= 0 ? __ldg(p + c[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < SU; ++u) if (c[u] >= 0) sum = __dadd_rn(sum, __dmul_rn(v[u], g[u]));
    }
    const double rn = rold - sum;
    r[row] = rn;
    if (F & 4) {
      double d0 = rn * rn, d1 = 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) { d0 += __shfl_xor_sync(0xffffffffu, d0, o); d1 += __shfl_xor_sync(0xffffffffu, d1, o); }
      if (lane == 0) { slpart[2 * s] = d0; slpart[2 * s + 1] = d1; }
    } else {
      acc += rn * rn;
    }
    s = nx;
  }
  if (acc == 1234.5) r[0] = acc;
}

// 24-bit column indices (round 3 question: do fewer stream bytes per entry move the L2 -> SM bound?):
// the low 16 bits of every index in a u16 SELL array and the high 8 bits in a u8 SELL array
// (3 bytes per entry instead of 4: 96 instead of 128 bytes per warp step).
__global__ void split_idx24(const int32_t* idx, uint16_t* lo, uint8_t* hi, long long n) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) { lo[t] = (uint16_t)(idx[t] & 0xFFFF); hi[t] = (uint8_t)(idx[t] >> 16); }
}
template <int SU>
__global__ void __launch_bounds__(1024, 1) k1c(const uint16_t* __restrict__ lo, const uint8_t* __restrict__ hi,
                                              const double* __restrict__ val, const double* __restrict__ p,
                                              double* __restrict__ r, int nslices) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s0 = (int)((long long)nslices * blockIdx.x / gridDim.x), s1 = (int)((long long)nslices * (blockIdx.x + 1) / gridDim.x);
  for (int s = s0 + warp; s < s1; s += 32) {
    const long long row = (long long)s * 32 + lane;
    const double rold = r[row];
    double sum = 0.0;
    const long long b = (long long)s * L * 32 + lane;
#pragma unroll
    for (int j0 = 0; j0 < L; j0 += SU) {
      int32_t c[SU]; double v[SU], g[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        unsigned a, h;
        asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=r"(a) : "l"(lo + b + (j0 + u) * 32));
        asm volatile("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=r"(h) : "l"(hi + b + (j0 + u) * 32));
        c[u] = (int32_t)(a | (h << 16));
        v[u] = lds_stream(val + b + (j0 + u) * 32);
      }
#pragma unroll
      for (int u = 0; u < SU; ++u) g[u] = __ldg(p + c[u]);
#pragma unroll
      for (int u = 0; u < SU; ++u) sum = __dadd_rn(sum, __dmul_rn(v[u], g[u]));
    }
    r[row] = rold - sum;
  }
}

// CTA-level TMA staging of the streams (round 3 question: do bulk copies, which do not go through
// the LSU / L1 request path, leave more of the SM's L2 request throughput to the gathers?). Each
// CTA's slice range is contiguous in the SELL arrays; one producer thread streams it in stages of
// SPS slices (idx and val blocks, two bulk copies per stage) into an NST-stage ring; consumer warp
// w takes slice w of each stage, reads its 12 indices and values from shared memory into
// registers, releases the stage, then issues its 12 gathers.
template <int NWC, int NST, int SUB>
__global__ void __launch_bounds__((NWC + 1) * 32, 1) k1t(const int32_t* __restrict__ idx, const double* __restrict__ val,
                                                        const double* __restrict__ p, double* __restrict__ r, int nslices,
                                                        uint64_t pol) {
  extern __shared__ __align__(128) unsigned char smraw[];
  constexpr int SPS = NWC;
  constexpr int IB = SPS * L * 32 * 4, VB = SPS * L * 32 * 8, SB = IB + VB;
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + NST * SB);
  uint64_t* empty = full + NST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s0 = (int)((long long)nslices * blockIdx.x / gridDim.x), s1 = (int)((long long)nslices * (blockIdx.x + 1) / gridDim.x);
  const int nst = (s1 - s0 + SPS - 1) / SPS;
  if (threadIdx.x == 0) {
    for (int k = 0; k < NST; ++k) { plss::mbar_init(&full[k], 1); plss::mbar_init(&empty[k], NWC); }
    plss::fence_mbar_init();
  }
  __syncthreads();
  if (warp == NWC) {
    if (lane == 0) {
      for (int t = 0; t < nst; ++t) {
        const int k = t % NST;
        if (t >= NST) plss::mbar_wait(&empty[k], ((t / NST) - 1) & 1);
        const int sa = s0 + t * SPS, sb = min(s1, sa + SPS);
        const unsigned ib = (unsigned)(sb - sa) * L * 32 * 4, vb = (unsigned)(sb - sa) * L * 32 * 8;
        plss::mbar_expect_tx(&full[k], ib + vb);
        plss::tma_load(smraw + k * SB, idx + (long long)sa * L * 32, ib, &full[k], pol);
        plss::tma_load(smraw + k * SB + IB, val + (long long)sa * L * 32, vb, &full[k], pol);
      }
    }
    return;
  }
  for (int t = 0; t < nst; ++t) {
    const int k = t % NST;
    const int s = s0 + t * SPS + warp;
    const long long row = (long long)s * 32 + lane;
    double rold = 0.0;
    if (s < s1) rold = r[row];
    plss::mbar_wait(&full[k], (t / NST) & 1);
    int32_t c[L]; double v[L];
    if (s < s1) {
      const int32_t* ip = reinterpret_cast<const int32_t*>(smraw + k * SB) + warp * L * 32 + lane;
      const double* vp = reinterpret_cast<const double*>(smraw + k * SB + IB) + warp * L * 32 + lane;
#pragma unroll
      for (int j = 0; j < L; ++j) { c[j] = ip[j * 32]; v[j] = vp[j * 32]; }
    }
    __syncwarp();
    if (lane == 0) plss::mbar_arrive(&empty[k]);
    if (s < s1) {
      double sum = 0.0;
#pragma unroll
      for (int j0 = 0; j0 < L; j0 += SUB) {
        double g[SUB];
#pragma unroll
        for (int u = 0; u < SUB; ++u) g[u] = __ldg(p + c[j0 + u]);
#pragma unroll
        for (int u = 0; u < SUB; ++u) sum = __dadd_rn(sum, __dmul_rn(v[j0 + u], g[u]));
      }
      r[row] = rold - sum;
    }
  }
}
__global__ void fill_sptr(int32_t* sptr, int n) { int i = blockIdx.x * blockDim.x + threadIdx.x; if (i <= n) sptr[i] = i * L; }


// 128-bit per-lane stream loads (the north star names 128-bit vectorised loads
// of the idx / val streams): slice layout with 4 steps of a lane's indices in one int4 and 2 steps
// of its values in one double2 (lane l, steps 4q..4q+3 at idx4[(s*L/4 + q)*32 + l]).
__global__ void relayout_v(const int32_t* idx, const double* val, int4* idx4, double2* val2, int nslices) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)nslices * 32) return;
  const long long s = t / 32, l = t % 32;
  for (int q = 0; q < L / 4; ++q) {
    int4 v;
    v.x = idx[(s * L + 4 * q + 0) * 32 + l]; v.y = idx[(s * L + 4 * q + 1) * 32 + l];
    v.z = idx[(s * L + 4 * q + 2) * 32 + l]; v.w = idx[(s * L + 4 * q + 3) * 32 + l];
    idx4[(s * (L / 4) + q) * 32 + l] = v;
  }
  for (int q = 0; q < L / 2; ++q) {
    double2 v;
    v.x = val[(s * L + 2 * q) * 32 + l]; v.y = val[(s * L + 2 * q + 1) * 32 + l];
    val2[(s * (L / 2) + q) * 32 + l] = v;
  }
}
__device__ __forceinline__ int4 ldi4_stream(const int4* p) {
  int4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p)); return v;
}
__device__ __forceinline__ double2 ldd2_stream(const double2* p) {
  double2 v; asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p)); return v;
}
__global__ void __launch_bounds__(1024, 1) k1v(const int4* __restrict__ idx4, const double2* __restrict__ val2,
                                              const double* __restrict__ p, double* __restrict__ r, int nslices) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s0 = (int)((long long)nslices * blockIdx.x / gridDim.x), s1 = (int)((long long)nslices * (blockIdx.x + 1) / gridDim.x);
  for (int s = s0 + warp; s < s1; s += 32) {
    const long long row = (long long)s * 32 + lane;
    const double rold = r[row];
    double sum = 0.0;
#pragma unroll
    for (int h = 0; h < L / 6; ++h) {                     // two batches of 6 steps
      int c[6]; double v[6], g[6];
      const int4 a0 = ldi4_stream(idx4 + ((long long)s * (L / 4) + 3 * h / 2) * 32 + lane);
      (void)a0;
#pragma unroll
      for (int u = 0; u < 6; ++u) {
        const int j = 6 * h + u;
        const int4 q4 = ldi4_stream(idx4 + ((long long)s * (L / 4) + j / 4) * 32 + lane);
        c[u] = (j & 3) == 0 ? q4.x : (j & 3) == 1 ? q4.y : (j & 3) == 2 ? q4.z : q4.w;
      }
#pragma unroll
      for (int u = 0; u < 6; u += 2) {
        const double2 d2 = ldd2_stream(val2 + ((long long)s * (L / 2) + (6 * h + u) / 2) * 32 + lane);
        v[u] = d2.x; v[u + 1] = d2.y;
      }
#pragma unroll
      for (int u = 0; u < 6; ++u) g[u] = __ldg(p + c[u]);
#pragma unroll
      for (int u = 0; u < 6; ++u) sum = __dadd_rn(sum, __dmul_rn(v[u], g[u]));
    }
    r[row] = rold - sum;
  }
}
// the same with all 12 indices from 3 int4 loads and 12 values from 6 double2 loads up front
__global__ void __launch_bounds__(1024, 1) k1v12(const int4* __restrict__ idx4, const double2* __restrict__ val2,
                                                const double* __restrict__ p, double* __restrict__ r, int nslices) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s0 = (int)((long long)nslices * blockIdx.x / gridDim.x), s1 = (int)((long long)nslices * (blockIdx.x + 1) / gridDim.x);
  for (int s = s0 + warp; s < s1; s += 32) {
    const long long row = (long long)s * 32 + lane;
    const double rold = r[row];
    int4 q[3]; double2 d[6];
#pragma unroll
    for (int k = 0; k < 3; ++k) q[k] = ldi4_stream(idx4 + ((long long)s * 3 + k) * 32 + lane);
#pragma unroll
    for (int k = 0; k < 6; ++k) d[k] = ldd2_stream(val2 + ((long long)s * 6 + k) * 32 + lane);
    const int c[12] = {q[0].x, q[0].y, q[0].z, q[0].w, q[1].x, q[1].y, q[1].z, q[1].w, q[2].x, q[2].y, q[2].z, q[2].w};
    double g[12];
#pragma unroll
    for (int u = 0; u < 12; ++u) g[u] = __ldg(p + c[u]);
    double sum = 0.0;
#pragma unroll
    for (int u = 0; u < 12; ++u) sum = __dadd_rn(sum, __dmul_rn(u & 1 ? d[u / 2].y : d[u / 2].x, g[u]));
    r[row] = rold - sum;
  }
}

// Split layout: band part (6 steps) from the shared-memory window, uniform part (6 steps) from
// global memory; no per-lane branch.
template <int BS>
__global__ void __launch_bounds__(BS, 1) k1_split(const int32_t* __restrict__ bidx, const double* __restrict__ bval,
                                                  const int32_t* __restrict__ uidx, const double* __restrict__ uval,
                                                  const double* __restrict__ p, double* __restrict__ r, int nslices, int chunk,
                                                  int band_smem) {
  extern __shared__ double sp[];
  constexpr int NW = BS / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s0 = (int)((long long)nslices * blockIdx.x / gridDim.x), s1 = (int)((long long)nslices * (blockIdx.x + 1) / gridDim.x);
  for (int c0 = s0; c0 < s1; c0 += chunk) {
    const int c1 = min(s1, c0 + chunk);
    const long long wlo = band_lo(OFF + (long long)c0 * 32), whi = band_lo(OFF + (long long)c1 * 32 - 1) + 2049;
    if (band_smem) {
      __syncthreads();
      for (long long q = wlo + threadIdx.x; q < whi; q += BS) sp[q - wlo] = __ldg(p + q);
      __syncthreads();
    }
    for (int s = c0 + warp; s < c1; s += NW) {
      const long long row = (long long)s * 32 + lane;
      double sum = 0.0;
      {
        int32_t c[NB]; double v[NB], g[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) { c[u] = ldi_stream(bidx + ((long long)s * NB + u) * 32 + lane); v[u] = lds_stream(bval + ((long long)s * NB + u) * 32 + lane); }
#pragma unroll
        for (int u = 0; u < NB; ++u) g[u] = band_smem ? sp[c[u] - wlo] : __ldg(p + c[u]);
#pragma unroll
        for (int u = 0; u < NB; ++u) sum = __dadd_rn(sum, __dmul_rn(v[u], g[u]));
      }
      {
        int32_t c[L - NB]; double v[L - NB], g[L - NB];
#pragma unroll
        for (int u = 0; u < L - NB; ++u) { c[u] = ldi_stream(uidx + ((long long)s * (L - NB) + u) * 32 + lane); v[u] = lds_stream(uval + ((long long)s * (L - NB) + u) * 32 + lane); }
#pragma unroll
        for (int u = 0; u < L - NB; ++u) g[u] = __ldg(p + c[u]);
#pragma unroll
        for (int u = 0; u < L - NB; ++u) sum = __dadd_rn(sum, __dmul_rn(v[u], g[u]));
      }
      r[row] = r[row] - sum;
    }
  }
}

// ---- K2 band part: the slab's band columns j in [J0, J0 + NJ), 48 band rows each in
// [8j - 8192, 8j + 8192) (slab rows only), sorted. CSC (column j's entries contiguous) and SELL.
constexpr int NJ = RS / 8;                  // 800k columns whose band centre lies in the slab
constexpr long long J0 = OFF / 8;
constexpr int KB = 48;
__global__ void gen_k2(int32_t* cidx, double* cval, int32_t* sidx, double* sval) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= NJ) return;
  const long long j = J0 + t;
  long long lo = 8 * j - 8192, hi = 8 * j + 8192;
  if (lo < OFF) lo = OFF;
  if (hi > OFF + RS) hi = OFF + RS;
  int32_t rr[KB];
  uint64_t h = mix(j * 104729ull);
  for (int k = 0; k < KB; ++k) {
    for (;;) {
      h = mix(h);
      const int32_t cand = (int32_t)(lo + (long long)(h % (uint64_t)(hi - lo)) - OFF);  // slab-local row
      bool dup = false;
      for (int q = 0; q < k; ++q) dup |= rr[q] == cand;
      if (!dup) { rr[k] = cand; break; }
    }
  }
  for (int a = 0; a < KB; ++a) for (int b = a + 1; b < KB; ++b) if (rr[b] < rr[a]) { int32_t x = rr[a]; rr[a] = rr[b]; rr[b] = x; }
  const long long s = t / 32, l = t % 32;
  for (int k = 0; k < KB; ++k) {
    h = mix(h);
    const double v = (double)(h % 2000001) * 1e-6 - 1.0;
    cidx[t * KB + k] = rr[k]; cval[t * KB + k] = v;
    sidx[(s * KB + k) * 32 + l] = rr[k]; sval[(s * KB + k) * 32 + l] = v;
  }
}

// lane per column (SELL), gathers from global r (what libplss does today)
template <int SU>
__global__ void __launch_bounds__(1024, 1) k2_sell(const int32_t* __restrict__ idx, const double* __restrict__ val,
                                                   const double* __restrict__ r, double* __restrict__ y) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nsl = NJ / 32;
  const int s0 = (int)((long long)nsl * blockIdx.x / gridDim.x), s1 = (int)((long long)nsl * (blockIdx.x + 1) / gridDim.x);
  for (int s = s0 + warp; s < s1; s += 32) {
    double sum = 0.0;
    for (int j0 = 0; j0 < KB; j0 += SU) {
      int32_t c[SU]; double v[SU], g[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) { c[u] = ldi_stream(idx + ((long long)s * KB + j0 + u) * 32 + lane); v[u] = lds_stream(val + ((long long)s * KB + j0 + u) * 32 + lane); }
#pragma unroll
      for (int u = 0; u < SU; ++u) g[u] = __ldg(r + c[u]);
#pragma unroll
      for (int u = 0; u < SU; ++u) sum = __dadd_rn(sum, __dmul_rn(v[u], g[u]));
    }
    y[(long long)s * 32 + lane] = sum;
  }
}

// warp per column (lanes over the column's 48 entries, fixed butterfly), r from global memory or
// from a shared-memory window of the CTA's current column chunk (loaded per chunk)
template <bool SMEM>
__global__ void __launch_bounds__(1024, 1) k2_wpc(const int32_t* __restrict__ idx, const double* __restrict__ val,
                                                  const double* __restrict__ r, double* __restrict__ y, int chunk) {
  extern __shared__ double sr[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = (int)((long long)NJ * blockIdx.x / gridDim.x), t1 = (int)((long long)NJ * (blockIdx.x + 1) / gridDim.x);
  for (int c0 = t0; c0 < t1; c0 += chunk) {
    const int c1 = min(t1, c0 + chunk);
    long long wlo = 8 * (J0 + c0) - 8192 - OFF, whi = 8 * (J0 + c1) + 8192 - OFF;
    if (wlo < 0) wlo = 0;
    if (whi > RS) whi = RS;
    if (SMEM) {
      __syncthreads();
      for (long long q = wlo + threadIdx.x; q < whi; q += 1024) sr[q - wlo] = __ldg(r + q);
      __syncthreads();
    }
    for (int t = c0 + warp; t < c1; t += 32) {
      const int32_t a0 = ldi_stream(idx + (long long)t * KB + lane);
      const double v0 = lds_stream(val + (long long)t * KB + lane);
      int32_t a1 = 0; double v1 = 0.0;
      if (lane < KB - 32) { a1 = ldi_stream(idx + (long long)t * KB + 32 + lane); v1 = lds_stream(val + (long long)t * KB + 32 + lane); }
      double g0 = SMEM ? sr[a0 - wlo] : __ldg(r + a0);
      double g1 = lane < KB - 32 ? (SMEM ? sr[a1 - wlo] : __ldg(r + a1)) : 0.0;
      double s = v0 * g0 + v1 * g1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) y[t] = s;
    }
  }
}

__global__ void fillv(double* x, long long n, double v) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) x[i] = v + (double)(i % 7);
}
__global__ void stream_copy(const double* a, double* b, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) b[i] = a[i];
}

template <class F>
float timeit(F f, int reps = 5) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  f();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const long long nnz = (long long)RS * L;
  int32_t *idx, *bidx, *uidx; double *val, *bval, *uval, *p, *r, *big;
  CK(cudaMalloc(&idx, nnz * 4)); CK(cudaMalloc(&val, nnz * 8));
  CK(cudaMalloc(&bidx, nnz / 2 * 4)); CK(cudaMalloc(&bval, nnz / 2 * 8));
  CK(cudaMalloc(&uidx, nnz / 2 * 4)); CK(cudaMalloc(&uval, nnz / 2 * 8));
  CK(cudaMalloc(&p, N * 8)); CK(cudaMalloc(&r, (long long)RS * 8));
  CK(cudaMalloc(&big, 1ll << 30));
  fillv<<<1024, 256>>>(p, N, 0.5); fillv<<<1024, 256>>>(r, RS, 0.25);
  gen_k1<<<(RS + 255) / 256, 256>>>(idx, val, bidx, bval, uidx, uval);
  CK(cudaDeviceSynchronize());
  {
    const long long nn = (1ll << 30) / 16;
    float ms = timeit([&] { stream_copy<<<sms * 8, 256>>>(big, big + nn, nn); });
    printf("copy 512 MB -> 512 MB: %.1f GB/s\n", 2.0 * nn * 8 / (ms / 1e3) / 1e9);
  }
  const double k1_bytes = nnz * 12.0 + RS * 16.0 + N * 8.0 / 10;   // stream + r RMW (+ p share)
  auto rep = [&](const char* name, float ms, double bytes, long long gathers) {
    printf("%-58s %7.3f ms  %6.0f GB/s  %.3f gathers/clk/SM (at %d MHz)\n", name, ms, bytes / (ms / 1e3) / 1e9,
           gathers / (ms / 1e3) / sms / (clk * 1e3), clk / 1000);
  };
  const int nsl = RS / 32;
  auto K1 = [&](auto kern, int bs, int grid, int smem, int chunk) {
    if (smem) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    return timeit([&] { kern<<<grid, bs, smem>>>(idx, val, p, r, nsl, chunk); });
  };
  printf("== K1 slab: %d rows x %d entries (6 band + 6 uniform), SELL-32\n", RS, L);
  if (getenv("BB_TMA")) {
    uint64_t pol_first;
    {
      uint64_t* d_pol; CK(cudaMalloc(&d_pol, 16));
      plss::k_policies<<<1, 1>>>(d_pol);
      uint64_t pols[2]; CK(cudaMemcpy(pols, d_pol, 16, cudaMemcpyDeviceToHost));
      pol_first = pols[0];
    }
    auto T = [&](auto kern, int nwc, int nst, const char* nm) {
      const int smem = nst * nwc * L * 32 * 12 + 2 * nst * 8;
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      rep(nm, timeit([&] { kern<<<sms, (nwc + 1) * 32, smem>>>(idx, val, p, r, nsl, pol_first); }), k1_bytes, nnz);
      CK(cudaGetLastError());
    };
    for (int rep_ = 0; rep_ < 2; ++rep_) {
      rep("K1 plain 32-bit idx (SU 6)", K1(k1<0, 1024, 6>, 1024, sms, 0, 0), k1_bytes, nnz);
      T(k1t<8, 2, 12>, 8, 2, "K1 TMA streams 8 warps x 2 stages (36 KB), 12 gathers");
      T(k1t<8, 3, 12>, 8, 3, "K1 TMA streams 8 warps x 3 stages (36 KB), 12 gathers");
      T(k1t<4, 2, 12>, 4, 2, "K1 TMA streams 4 warps x 2 stages (18 KB), 12 gathers");
      T(k1t<4, 4, 12>, 4, 4, "K1 TMA streams 4 warps x 4 stages (18 KB), 12 gathers");
      T(k1t<2, 4, 12>, 2, 4, "K1 TMA streams 2 warps x 4 stages (9 KB), 12 gathers");
      T(k1t<8, 4, 12>, 8, 4, "K1 TMA streams 8 warps x 4 stages (36 KB), 12 gathers");
      T(k1t<16, 2, 12>, 16, 2, "K1 TMA streams 16 warps x 2 stages (72 KB), 12 gathers");
      T(k1t<4, 8, 12>, 4, 8, "K1 TMA streams 4 warps x 8 stages (18 KB), 12 gathers");
    }
    if (getenv("BB_ONLY")) return 0;
  }
  if (getenv("BB_IDX24")) {
    uint16_t* lo; uint8_t* hi;
    CK(cudaMalloc(&lo, nnz * 2)); CK(cudaMalloc(&hi, nnz));
    split_idx24<<<(unsigned)((nnz + 255) / 256), 256>>>(idx, lo, hi, nnz);
    CK(cudaDeviceSynchronize());
    for (int rep_ = 0; rep_ < 3; ++rep_) {
      rep("K1 plain 32-bit idx (SU 6)", K1(k1<0, 1024, 6>, 1024, sms, 0, 0), k1_bytes, nnz);
      rep("K1 24-bit idx u16+u8 (SU 6)", timeit([&] { k1c<6><<<sms, 1024>>>(lo, hi, val, p, r, nsl); }), k1_bytes, nnz);
      rep("K1 24-bit idx u16+u8 (SU 12)", timeit([&] { k1c<12><<<sms, 1024>>>(lo, hi, val, p, r, nsl); }), k1_bytes, nnz);
      rep("K1 no gathers (SU 6)", K1(k1<3, 1024, 6>, 1024, sms, 0, 0), k1_bytes, 0);
    }
    CK(cudaFree(lo)); CK(cudaFree(hi));
    if (getenv("BB_ONLY")) return 0;
  }
  rep("K1 full (1024 x 1/SM, SU 6)", K1(k1<0, 1024, 6>, 1024, sms, 0, 0), k1_bytes, nnz);
  rep("K1 full (1024 x 1/SM, SU 12)", K1(k1<0, 1024, 12>, 1024, sms, 0, 0), k1_bytes, nnz);
  rep("K1 full (512 x 2/SM, SU 6)", K1(k1<0, 512, 6>, 512, 2 * sms, 0, 0), k1_bytes, nnz);
  rep("K1 full (256 x 8/SM, SU 4)", K1(k1<0, 256, 4>, 256, 8 * sms, 0, 0), k1_bytes, nnz);
  rep("K1 band gathers skipped (SU 6)", K1(k1<1, 1024, 6>, 1024, sms, 0, 0), k1_bytes, nnz / 2);
  rep("K1 uniform gathers skipped (SU 6)", K1(k1<2, 1024, 6>, 1024, sms, 0, 0), k1_bytes, nnz / 2);
  rep("K1 band ldg, uniform ld.cg (SU 6)", K1(k1<6, 1024, 6>, 1024, sms, 0, 0), k1_bytes, nnz);
  rep("K1 band ldg, uniform ld.cg (SU 12)", K1(k1<6, 1024, 12>, 1024, sms, 0, 0), k1_bytes, nnz);
  rep("K1 band ldg, uniform L1::no_allocate (SU 6)", K1(k1<7, 1024, 6>, 1024, sms, 0, 0), k1_bytes, nnz);
  rep("K1 all gathers ld.cg (SU 6)", K1(k1<8, 1024, 6>, 1024, sms, 0, 0), k1_bytes, nnz);
  rep("K1 band ldg, uniform ld.cs (SU 6)", K1(k1<9, 1024, 6>, 1024, sms, 0, 0), k1_bytes, nnz);
  rep("K1 no gathers (SU 6)", K1(k1<3, 1024, 6>, 1024, sms, 0, 0), k1_bytes, 0);
  rep("K1 no streams, gathers only (SU 6)", K1(k1<5, 1024, 6>, 1024, sms, 0, 0), RS * 16.0, nnz);

  {
    rep("K1 plain, r_old early (SU 6)", timeit([&] { k1e<6><<<sms, 1024>>>(idx, val, p, r, nsl); }), k1_bytes, nnz);
    rep("K1 plain, r_old early (SU 12)", timeit([&] { k1e<12><<<sms, 1024>>>(idx, val, p, r, nsl); }), k1_bytes, nnz);
    auto P = [&](auto kern, int bs, int grid, int smem, const char* nm) {
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      rep(nm, timeit([&] { kern<<<grid, bs, smem>>>(idx, val, p, r, nsl); }), k1_bytes, nnz);
    };
    if (getenv("BB_ALL")) P(k1p<4, 4, 1024>, 1024, sms, 32 * 4 * 4 * 384, "K1 cp.async ring SUB 4 NSTG 4 (1024 x 1)");
    if (getenv("BB_ALL")) P(k1p<4, 3, 1024>, 1024, sms, 32 * 3 * 4 * 384, "K1 cp.async ring SUB 4 NSTG 3 (1024 x 1)");
    if (getenv("BB_ALL")) P(k1p<3, 5, 1024>, 1024, sms, 32 * 5 * 3 * 384, "K1 cp.async ring SUB 3 NSTG 5 (1024 x 1)");
    if (getenv("BB_ALL")) P(k1p<2, 8, 1024>, 1024, sms, 32 * 8 * 2 * 384, "K1 cp.async ring SUB 2 NSTG 8 (1024 x 1)");
    if (getenv("BB_ALL")) P(k1p<6, 2, 1024>, 1024, sms, 32 * 2 * 6 * 384, "K1 cp.async ring SUB 6 NSTG 2 (1024 x 1)");
    if (getenv("BB_ALL")) P(k1p<4, 4, 512>, 512, 2 * sms, 16 * 4 * 4 * 384, "K1 cp.async ring SUB 4 NSTG 4 (512 x 2)");
    if (getenv("BB_ALL")) P(k1p<2, 4, 512>, 512, 2 * sms, 16 * 4 * 2 * 384, "K1 cp.async ring SUB 2 NSTG 4 (512 x 2)");
  }

  {
    int32_t* sptr; double* slpart;
    CK(cudaMalloc(&sptr, (nsl + 1) * 4)); CK(cudaMalloc(&slpart, nsl * 16));
    fill_sptr<<<(nsl + 256) / 256, 256>>>(sptr, nsl);
    CK(cudaDeviceSynchronize());
    auto X = [&](auto kern, const char* nm) { rep(nm, timeit([&] { kern<<<sms, 1024>>>(idx, val, p, r, nsl, sptr, slpart); }), k1_bytes, nnz); };
    X(k1x<0>, "K1x plain (static, SU 6, register rho)");
    X(k1x<1>, "K1x + dynamic tickets");
    X(k1x<2>, "K1x + sptr loads");
    X(k1x<4>, "K1x + per-slice rho partials");
    X(k1x<8>, "K1x + evict-first streams");
    X(k1x<16>, "K1x + SU 8 with predicated tail");
    X(k1x<31>, "K1x all (libplss-like)");
    X(k1x<15>, "K1x all but SU 8");
    X(k1x<23>, "K1x all but evict-first");
    CK(cudaFree(sptr)); CK(cudaFree(slpart));
  }

  {
    // the production kernel (libplss k_sell<ROLE_K1, 1024, ..., STAT>) on the same slab
    int32_t *sptr, *cblk; double *slpart, *part; unsigned* cnt;
    CK(cudaMalloc(&sptr, (nsl + 1) * 4)); CK(cudaMalloc(&slpart, nsl * 16)); CK(cudaMalloc(&cblk, 4096 * 4));
    CK(cudaMalloc(&part, 4096 * 16)); CK(cudaMalloc(&cnt, 64));
    fill_sptr<<<(nsl + 256) / 256, 256>>>(sptr, nsl);
    const int nblocks = (nsl + 15) / 16;
    plss::k_cta_ranges<<<1, 256>>>(sptr, 32, nsl, 16, nblocks, sms, cblk, 128);
    CK(cudaDeviceSynchronize());
    plss::SpmvSeg a; memset(&a, 0, sizeof a);
    a.idx = idx; a.val = val; a.nrows = RS; a.g = p; a.out = r; a.partial = part; a.part_base = part; a.nparts = sms;
    a.counter = cnt; a.fmt = 3; a.nslices = nsl; a.sptr = sptr; a.cblk = cblk; a.slpart = slpart; a.stat = 1;
    {
      uint64_t* d_pol; CK(cudaMalloc(&d_pol, 16));
      plss::k_policies<<<1, 1>>>(d_pol);
      uint64_t pols[2]; CK(cudaMemcpy(pols, d_pol, 16, cudaMemcpyDeviceToHost));
      a.pol_first = pols[0]; a.pol_last = pols[1];
    }
    rep("libplss k_sell<K1,1024> dynamic", timeit([&] { plss::k_sell<plss::ROLE_K1, 1024><<<sms, 1024>>>(a); }), k1_bytes, nnz);
    rep("libplss k_sell<K1,1024,STAT>", timeit([&] { plss::k_sell<plss::ROLE_K1, 1024, false, false, plss::SIGMA, true><<<sms, 1024>>>(a); }), k1_bytes, nnz);
    a.pol_first = 0;
    rep("libplss k_sell<K1,1024,STAT> policy 0", timeit([&] { plss::k_sell<plss::ROLE_K1, 1024, false, false, plss::SIGMA, true><<<sms, 1024>>>(a); }), k1_bytes, nnz);
    CK(cudaFree(sptr)); CK(cudaFree(slpart)); CK(cudaFree(cblk)); CK(cudaFree(part)); CK(cudaFree(cnt));
  }

  {
    int4* idx4; double2* val2;
    CK(cudaMalloc(&idx4, nnz * 4)); CK(cudaMalloc(&val2, nnz * 8));
    relayout_v<<<(nsl * 32 + 255) / 256, 256>>>(idx, val, idx4, val2, nsl);
    CK(cudaDeviceSynchronize());
    rep("K1 128-bit lanes: int4 idx + double2 val, batches of 6", timeit([&] { k1v<<<sms, 1024>>>(idx4, val2, p, r, nsl); }), k1_bytes, nnz);
    rep("K1 128-bit lanes: all 12 up front", timeit([&] { k1v12<<<sms, 1024>>>(idx4, val2, p, r, nsl); }), k1_bytes, nnz);
    rep("K1 plain (reference, SU 6)", K1(k1<0, 1024, 6>, 1024, sms, 0, 0), k1_bytes, nnz);
    CK(cudaFree(idx4)); CK(cudaFree(val2));
  }
  if (getenv("BB_ALL")) for (int ch : {64, 256, 1024}) {
    char nm[96];
    const int smem = ((ch * 32) / 8 + 2049 + 8) * 8;
    snprintf(nm, sizeof nm, "K1 band from smem window, mixed (1024x1, chunk %d sl)", ch);
    rep(nm, K1(k1<4, 1024, 6>, 1024, sms, smem, ch), k1_bytes, nnz);
    snprintf(nm, sizeof nm, "K1 band from smem window, mixed (512x2, chunk %d sl)", ch);
    rep(nm, K1(k1<4, 512, 6>, 512, 2 * sms, smem, ch), k1_bytes, nnz);
  }
  if (getenv("BB_ALL")) for (int ch : {256, 1024}) {
    const int smem = ((ch * 32) / 8 + 2049 + 8) * 8;
    CK(cudaFuncSetAttribute(k1_split<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(k1_split<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    char nm[96];
    snprintf(nm, sizeof nm, "K1 split, band from global (1024x1, chunk %d)", ch);
    rep(nm, timeit([&] { k1_split<1024><<<sms, 1024, smem>>>(bidx, bval, uidx, uval, p, r, nsl, ch, 0); }), k1_bytes, nnz);
    snprintf(nm, sizeof nm, "K1 split, band from smem (1024x1, chunk %d)", ch);
    rep(nm, timeit([&] { k1_split<1024><<<sms, 1024, smem>>>(bidx, bval, uidx, uval, p, r, nsl, ch, 1); }), k1_bytes, nnz);
    snprintf(nm, sizeof nm, "K1 split, band from smem (512x2, chunk %d)", ch);
    rep(nm, timeit([&] { k1_split<512><<<2 * sms, 512, smem>>>(bidx, bval, uidx, uval, p, r, nsl, ch, 1); }), k1_bytes, nnz);
  }
  CK(cudaFree(idx)); CK(cudaFree(val)); CK(cudaFree(bidx)); CK(cudaFree(bval)); CK(cudaFree(uidx)); CK(cudaFree(uval));

  printf("== K2 band half: %d columns x %d band rows (slab rows, window 16384 rows)\n", NJ, KB);
  const long long nk = (long long)NJ * KB;
  int32_t *cidx, *sidx; double *cval, *sval, *y;
  CK(cudaMalloc(&cidx, nk * 4)); CK(cudaMalloc(&cval, nk * 8)); CK(cudaMalloc(&sidx, nk * 4)); CK(cudaMalloc(&sval, nk * 8));
  CK(cudaMalloc(&y, NJ * 8));
  gen_k2<<<(NJ + 255) / 256, 256>>>(cidx, cval, sidx, sval);
  CK(cudaDeviceSynchronize());
  const double k2_bytes = nk * 12.0 + NJ * 8.0 + RS * 8.0;
  rep("K2 band, lane per column SELL (SU 8), r global", timeit([&] { k2_sell<8><<<sms, 1024>>>(sidx, sval, r, y); }), k2_bytes, nk);
  rep("K2 band, lane per column SELL (SU 12), r global", timeit([&] { k2_sell<12><<<sms, 1024>>>(sidx, sval, r, y); }), k2_bytes, nk);
  rep("K2 band, warp per column, r global", timeit([&] { k2_wpc<false><<<sms, 1024>>>(cidx, cval, r, y, 1 << 30); }), k2_bytes, nk);
  for (int ch : {256, 512, 1024, 2048}) {
    const int smem = (8 * ch + 16384 + 16) * 8;
    if (smem > 227 * 1024) continue;
    CK(cudaFuncSetAttribute(k2_wpc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    char nm[96];
    snprintf(nm, sizeof nm, "K2 band, warp per column, r smem window (chunk %d cols)", ch);
    rep(nm, timeit([&] { k2_wpc<true><<<sms, 1024, smem>>>(cidx, cval, r, y, ch); }), k2_bytes, nk);
  }
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}
