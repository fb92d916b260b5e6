// Peer-memory all-reduce of the distributed step (SURVEY 8(e) improvement 3; options.flags bit3).
//
// Row blocks: every rank holds a partial y_g = A_g^T r_g (and its local rho in
// element n); the step needs y = sum_g y_g on every rank. Instead of ncclAllReduce, each rank
// maps the other ranks' buffers (CUDA IPC, handles exchanged once at create) and, per column
// chunk of K2 -- on the communication stream while K2 computes the next chunk --
//   1. signals "my partial of chunk c is complete" into every peer's flag block,
//   2. waits until every rank signalled chunk c,
//   3. sums its column shard of the chunk over all ranks' partials in rank order 0..G-1 (loads
//      through NVLink) and stores the sum into every rank's reduced y (stores through NVLink),
//   4. the last CTA signals "chunk c of my shard is written" to every peer.
// k_peer_wait (main stream, before the dots kernel) waits for every rank's step-4 signal of every
// chunk, then advances the epoch. Each element is summed once, by its owner, in a fixed order and
// stored to all ranks, so y -- and every scalar and decision derived from it -- is bitwise
// identical on every rank (what ncclAllReduce guaranteed before).
//
// The flags carry the epoch (one per loop step; all ranks run the same steps), so they are never
// reset. Kernels no-op once ctl->done (identical on every rank). Spins are bounded: after
// PEER_TIMEOUT_NS the kernel records PF_ERR and stops waiting (the solve then reports an error
// instead of hanging the GPU).
//
// The rank is rank_base + blockIdx.y: a distributed ctx launches one grid row (its own rank); the
// single-GPU test entry point plss_peer_reduce_emulate launches G rows cooperatively over G sets
// of buffers, one per virtual rank (the same code, all ranks' data in one kernel).
#pragma once
#include <cstdint>

namespace plss {

constexpr int PEER_MAX = 8;        // ranks
constexpr int PEER_NCH = 8;        // column chunks (>= DCH_MAX)
constexpr int PEER_NT = 512;
// per-rank flag block (u32 words)
constexpr int PF_ARRIVE = 0;                                // [c][h]: rank h's partial of chunk c is complete
constexpr int PF_DONE = PEER_NCH * PEER_MAX;                // [c][h]: rank h wrote its shard of chunk c here
constexpr int PF_CNT = 2 * PEER_NCH * PEER_MAX;             // [c]: CTAs of this rank's reduce of chunk c
constexpr int PF_EP = PF_CNT + PEER_NCH;                    // steps completed
constexpr int PF_ERR = PF_EP + 1;                           // a wait timed out
constexpr int PF_WORDS = 256;
constexpr unsigned long long PEER_TIMEOUT_NS = 20ull * 1000 * 1000 * 1000;

struct PeerTab {
  const double* part[PEER_MAX];    // rank h's partial y | rho (K1 / K2 output), n + 1 doubles
  double* red[PEER_MAX];           // rank h's reduced y | rho
  unsigned* flg[PEER_MAX];         // rank h's flag block
};

__device__ __forceinline__ void peer_st_release(unsigned* a, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned peer_ld_acquire(const unsigned* a) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
// release fence at system scope (MEMBAR.ALL.SYS; __threadfence_system is the heavier SC fence)
__device__ __forceinline__ void peer_fence() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ unsigned long long peer_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// wait until *a has reached epoch E (flags only grow); false on timeout (PF_ERR set)
__device__ __forceinline__ bool peer_wait(const unsigned* a, unsigned E, unsigned* own) {
  if ((int)(peer_ld_acquire(a) - E) >= 0) return true;
  const unsigned long long t0 = peer_now();
  while ((int)(peer_ld_acquire(a) - E) < 0) {
    __nanosleep(64);
    if (peer_now() - t0 > PEER_TIMEOUT_NS) {
      atomicExch(own + PF_ERR, 1u);
      return false;
    }
  }
  return true;
}

__device__ __forceinline__ long long peer_min(long long a, long long b) { return a < b ? a : b; }

// sum over ranks in order 0..G-1 of element j, stored to every rank
template <int V>
__device__ __forceinline__ void peer_sum_store(const PeerTab& t, int G, long long j) {
  if constexpr (V == 2) {
    double2 v[PEER_MAX];
#pragma unroll
    for (int h = 0; h < PEER_MAX; ++h)
      if (h < G) v[h] = __ldcg(reinterpret_cast<const double2*>(t.part[h] + j));
    double2 s = v[0];
#pragma unroll
    for (int h = 1; h < PEER_MAX; ++h)
      if (h < G) { s.x = __dadd_rn(s.x, v[h].x); s.y = __dadd_rn(s.y, v[h].y); }
#pragma unroll
    for (int h = 0; h < PEER_MAX; ++h)
      if (h < G) __stcg(reinterpret_cast<double2*>(t.red[h] + j), s);
  } else {
    double v[PEER_MAX];
#pragma unroll
    for (int h = 0; h < PEER_MAX; ++h)
      if (h < G) v[h] = __ldcg(t.part[h] + j);
    double s = v[0];
#pragma unroll
    for (int h = 1; h < PEER_MAX; ++h)
      if (h < G) s = __dadd_rn(s, v[h]);
#pragma unroll
    for (int h = 0; h < PEER_MAX; ++h)
      if (h < G) __stcg(t.red[h] + j, s);
  }
}

// chunk c = elements [lo, hi) of y | rho; this rank's shard is the rank-th of G near-equal,
// even-aligned pieces
__global__ void __launch_bounds__(PEER_NT) k_peer_reduce(PeerTab t, int G, int rank_base, int c, long long lo,
                                                         long long hi, const Ctl* ctl) {
  if (ctl != nullptr && ctl->done) return;
  const int rank = rank_base + (int)blockIdx.y;
  unsigned* own = t.flg[rank];
  const unsigned E = *(volatile unsigned*)(own + PF_EP) + 1u;
  __shared__ int ok;
  if (threadIdx.x == 0) ok = 1;
  __syncthreads();
  // 1. arrive: CTA 0 signals that this rank's partial of chunk c is complete (the launch is
  //    stream-ordered after K2 of chunk c). The grid is sized to be co-resident with nothing but
  //    K2 (which finishes on its own) beside it, so CTAs spinning below cannot keep CTA 0 from
  //    running. 2. every CTA waits for every rank's arrival.
  if (blockIdx.x == 0 && threadIdx.x < (unsigned)G)
    peer_st_release(t.flg[threadIdx.x] + PF_ARRIVE + c * PEER_MAX + rank, E);
  if (threadIdx.x < (unsigned)G)
    if (!peer_wait(own + PF_ARRIVE + c * PEER_MAX + threadIdx.x, E, own)) ok = 0;
  __syncthreads();
  if (ok) {
    // 3. this rank's shard [s0, s1) of [lo, hi)
    const long long len = hi - lo;
    long long per = (len + G - 1) / G;
    per += per & 1;
    const long long s0 = peer_min(hi, lo + (long long)rank * per), s1 = peer_min(hi, s0 + per);
    const long long a0 = peer_min(s1, s0 + (s0 & 1));          // even start for the double2 part
    const long long a1 = a0 + ((s1 - a0) & ~1ll);
    const long long stride = (long long)gridDim.x * PEER_NT * 2;
    long long j = a0 + 2 * ((long long)blockIdx.x * PEER_NT + threadIdx.x);
    for (; j + stride < a1; j += 2 * stride) {              // 2 x G independent 16-byte loads in flight
      double2 v[2][PEER_MAX];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int h = 0; h < PEER_MAX; ++h)
          if (h < G) v[u][h] = __ldcg(reinterpret_cast<const double2*>(t.part[h] + j + u * stride));
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        double2 sm = v[u][0];
#pragma unroll
        for (int h = 1; h < PEER_MAX; ++h)
          if (h < G) { sm.x = __dadd_rn(sm.x, v[u][h].x); sm.y = __dadd_rn(sm.y, v[u][h].y); }
#pragma unroll
        for (int h = 0; h < PEER_MAX; ++h)
          if (h < G) __stcg(reinterpret_cast<double2*>(t.red[h] + j + u * stride), sm);
      }
    }
    for (; j < a1; j += stride) peer_sum_store<2>(t, G, j);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (a0 > s0) peer_sum_store<1>(t, G, s0);
      if (a1 < s1) peer_sum_store<1>(t, G, a1);
    }
  }
  // 4. the last CTA of this rank signals "shard of chunk c written" to every rank (the CTA's
  //    stores are ordered before thread 0's system-scope fence by the barrier, as in a grid sync)
  __syncthreads();
  if (threadIdx.x == 0) {
    peer_fence();
    const unsigned tk = atomicAdd(own + PF_CNT + c, 1u);
    if (tk == gridDim.x - 1) {
      own[PF_CNT + c] = 0u;                                   // next step starts from 0
      peer_fence();
      for (int h = 0; h < G; ++h) peer_st_release(t.flg[h] + PF_DONE + c * PEER_MAX + rank, E);
    }
  }
}

// every rank wrote its shard of every chunk into this rank's reduced y: advance the epoch
__global__ void k_peer_wait(PeerTab t, int G, int nch, int rank_base, const Ctl* ctl) {
  if (ctl != nullptr && ctl->done) return;
  const int rank = rank_base + (int)blockIdx.y;
  unsigned* own = t.flg[rank];
  const unsigned E = *(volatile unsigned*)(own + PF_EP) + 1u;
  const int i = threadIdx.x;
  if (i < nch * G) peer_wait(own + PF_DONE + (i / G) * PEER_MAX + (i % G), E, own);
  __syncthreads();
  if (i == 0) {
    own[PF_EP] = E;
    peer_fence();
  }
}

}  // namespace plss
