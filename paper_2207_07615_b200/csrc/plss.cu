// plss.cu -- host side of libplss: the C ABI declared in include/plss.h.
//
// One ctx = one matrix on one device (one row block on a rank). Device memory comes from the
// caller's workspace (torch); the library allocates only a few bytes of pinned host memory for
// the done flag. The solve loop runs as CUDA graphs of `chunk` iterations; each iteration is
//     for s in slabs: K1_s (r_s <- r_s - A_s p), K2_s (y += A_s^T r_s)     [2S launches]
//     [rank > 1: ncclAllReduce(y | rho, n+1), K2b (phi, psi, tails)]
//     K3 (p, x, theta)
// K1_s and K2_s alternate so the slab of r that K1_s just wrote is gathered by K2_s while it is
// still resident in L2.
#include "../../include/plss.h"
#include "plss_kernels.cuh"
#include "rp_kernels.cuh"
#include "kz_kernels.cuh"
#include "eg_kernels.cuh"
#include "peer_kernels.cuh"

#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <chrono>
#include <thread>
#include <vector>

// NVTX range around a host entry point or a graph chunk (tracing): a no-op unless
// a tool (nsys, ncu --nvtx) is attached. The loop's kernels run inside CUDA graphs, so the ranges
// mark the host calls and each chunk launch; kernels are told apart by name.
namespace {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace

using namespace plss;

namespace {

constexpr int MAXG = 2048;           // upper bound on persistent-CTA grid sizes (partials)
constexpr int DCH_MAX = 8;           // column chunks of the last K2 segment on a distributed ctx
static_assert(DCH_MAX <= PEER_NCH, "peer flag blocks cover every chunk");
constexpr int64_t DPAD = 64 * 32;    // vector slack for the reduce-scatter step (64 ranks x 32)
constexpr int SCAN_ITEMS = 16;       // setup scan: items per thread
constexpr size_t ALIGN = 256;

std::string g_last_error;

size_t align_up(size_t v) { return (v + ALIGN - 1) / ALIGN * ALIGN; }

int auto_slabs(int64_t m) {
  const char* env = std::getenv("PLSS_SLABS");
  if (env && std::atoi(env) > 0) return std::atoi(env);
  // r slab kept L2-resident between K1_s and K2_s; more slabs cost a y read-modify-write each.
  // C5 (512 MB of r), ms per step over 3 interleaved runs: 8 slabs 6.05-6.07, 9 5.96-5.97,
  // 10 5.93-5.94, 11 5.98-6.01, 12 6.09-6.11, 16 6.48 (scripts/gpu_slabs.sh); re-checked on the
  // final round-2 build, two interleaved runs: 8 5.48-5.49, 9 5.43-5.44, 10 5.42, 11 5.49
  const int64_t slab_bytes = 52ll << 20;
  int64_t s = (m * 8 + slab_bytes - 1) / slab_bytes;
  return (int)std::max<int64_t>(1, std::min<int64_t>(s, 64));
}

[[maybe_unused]] int64_t ntiles_of(int64_t nnz_s) { return std::max<int64_t>(1, (nnz_s + TILE - 1) / TILE); }

struct Layout {
  int S = 1;
  bool dist = false;
  int maxit_cap = 0;
  size_t wi;
  size_t r, y, p, x, rec, ctl, counters, part1, part2, part3, partn, tile1, tile2, scratch,
      scratch_blk, sptr, sidx, sval, scan_cnt, scan_blk, buf, err, scalars, total;
  bool sell = true;
  size_t s1idx, s1val, s1perm, s1sptr, s2idx, s2val, s2perm, s2sptr, s1win, s2win, cblk, slpart;
  size_t s1aux, s2aux;           // globally sorted segments: long-row lists + unit-weight prefixes
  int64_t s1auxn, s2auxn;
  bool window = true;
  int64_t s1cap, s2cap, s1slots, s2slots, s1sp, s2sp;  // pool capacities (entries / slots / sptr)
};

bool compute_layout(const plss_matrix* A, const plss_options* opt, bool dist, Layout* L) {
  if (!A || A->m < 0 || A->n < 0 || A->nnz < 0 || A->nnz >= (1ll << 31)) return false;
  plss_options o{};
  if (opt) o = *opt;
  int S = o.slabs > 0 ? o.slabs : auto_slabs(A->m);
  if (A->m > 0) S = (int)std::min<int64_t>(S, A->m);
  S = std::max(1, std::min(S, 64));
  L->S = S;
  L->dist = dist;
  L->maxit_cap = o.maxit_cap > 0 ? o.maxit_cap : 20000;
  const int64_t m = A->m, n = A->n, nnz = A->nnz;
  const int64_t tiles1 = nnz / TILE + m / RCAP + 2 * S + 2;       // K1 tile descriptors
  const int64_t tiles2 = nnz / TILE + S * (n / RCAP) + 2 * S + 2; // K2 tile descriptors
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o2 = off; off = align_up(off + std::max<size_t>(bytes, 1)); return o2; };
  L->r = take(8 * (m + 2));          // r[m]: theta partial of the column-block step
  // dist: y | rho (the all-reduce buffer); DPAD slack lets the reduce-scatter step pad y, p, x to
  // nranks x (32-aligned shard) doubles for up to 64 ranks
  L->y = take(8 * (n + 1 + DPAD));
  L->p = take(8 * (n + DPAD));
  L->x = take(8 * (n + DPAD));
  L->rec = take(8 * (size_t)(L->maxit_cap + 1) * REC);
  L->ctl = take(sizeof(Ctl));
  L->counters = take(64 * sizeof(unsigned));
  L->part1 = take(16 * (size_t)MAXG * S);
  L->part2 = take(16 * (size_t)MAXG);
  L->part3 = take(16 * (size_t)MAXG);
  L->partn = take(16 * (size_t)MAXG);
  L->tile1 = take(8 * (size_t)(tiles1 + S));
  L->tile2 = take(8 * (size_t)(tiles2 + S));
  L->scratch = take(4 * (size_t)(std::max(m, n) + 2));
  // SELL-32 pools (K1 over the CSR row slabs, K2 over the CSC slabs); opt.flags bit0 disables
  L->sell = !(o.flags & 1);
  if (L->sell) {
    L->s1cap = nnz * 115 / 100 + 4096ll * S;
    L->s2cap = nnz * 115 / 100 + 4096ll * S;
    L->s1slots = (m / 32 + 2 * S + 1) * 32;
    L->s2slots = (int64_t)S * (n / 32 + 2) * 32;
    L->s1sp = m / 32 + 3 * S + 2;
    L->s2sp = (int64_t)S * (n / 32 + 3) + 2;
    L->s1idx = take(4 * (size_t)L->s1cap);
    L->s1val = take(8 * (size_t)L->s1cap);
    L->s1perm = take(4 * (size_t)L->s1slots);
    L->s1sptr = take(4 * (size_t)L->s1sp);
    L->s2idx = take(4 * (size_t)L->s2cap);
    L->s2val = take(8 * (size_t)L->s2cap);
    L->s2perm = take(4 * (size_t)L->s2slots);
    L->s2sptr = take(4 * (size_t)L->s2sp);
    // window blocks (NSB slices each) of the windowed SELL segments; opt.flags bit1 disables
    L->window = !(o.flags & 2);
    L->s1win = take(8 * (size_t)(L->s1sp / 4 + 2 * S + 2));     // window blocks: nsb >= 4 slices
    L->s2win = take(8 * (size_t)(L->s2sp / 4 + 2 * S + 2));
    L->cblk = take(4 * (size_t)(MAXG + 1) * (2 * S + DCH_MAX));
    // units of one segment: slices + long rows (<= nnz / (LONGROW + 1) of them)
    L->slpart = take(16 * (size_t)(std::max(m, n) / 32 + nnz / (LONGROW + 1) + 4));
    L->s1auxn = 2 * (m / 32 + 4 * S + 8) + 8 * (nnz / (LONGROW + 1) + 2);
    L->s2auxn = 2 * ((int64_t)S * (n / 32) + 4 * S + 8) + 8 * (nnz / (LONGROW + 1) + 2);
    L->s1aux = take(4 * (size_t)L->s1auxn);
    L->s2aux = take(4 * (size_t)L->s2auxn);
  }
  L->scratch_blk = take(4 * (size_t)((std::max(m, n) + 2) / (NT * SCAN_ITEMS) + 2));
  if (S > 1) {
    // the slab-major CSC: in the workspace without SELL-32; with it, a setup-time allocation that
    // is released once every K2 segment streams its own SELL copy (setup, "slab-major CSC")
    if (!L->sell) {
      L->sptr = take(4 * (size_t)S * (n + 1));
      L->sidx = take(4 * (size_t)nnz);
      L->sval = take(8 * (size_t)nnz);
    } else {
      L->sptr = L->sidx = L->sval = 0;
    }
    L->scan_cnt = take(4 * (size_t)(n + 1));
    L->scan_blk = take(4 * (size_t)((n + 1) / (NT * SCAN_ITEMS) + 2));
  } else {
    L->sptr = L->sidx = L->sval = L->scan_cnt = L->scan_blk = 0;
  }
  L->buf = L->y;
  L->wi = take(8 * (size_t)(n + 1));   // PLSS W: the diagonal of WI (16-byte reads in K3)
  L->err = take(64);
  L->scalars = take(128);
  L->total = off;
  return true;
}

// ---- setup scan (exclusive, int32, deterministic; one-time) --------------------------------
__global__ void k_scan_local(int32_t* a, long long len, int32_t* blk) {
  __shared__ int32_t tsum[NT];
  const long long base = ((long long)blockIdx.x * NT + threadIdx.x) * SCAN_ITEMS;
  int32_t s = 0;
  for (int u = 0; u < SCAN_ITEMS; ++u) {
    const long long i = base + u;
    if (i < len) { const int32_t v = a[i]; a[i] = s; s += v; }
  }
  tsum[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t acc = 0;
    for (int t = 0; t < NT; ++t) { const int32_t v = tsum[t]; tsum[t] = acc; acc += v; }
    blk[blockIdx.x] = acc;
  }
  __syncthreads();
  const int32_t off = tsum[threadIdx.x];
  for (int u = 0; u < SCAN_ITEMS; ++u) {
    const long long i = base + u;
    if (i < len) a[i] += off;
  }
}
__global__ void k_scan_blocks(int32_t* blk, int nb) {
  int32_t acc = 0;
  for (int b = 0; b < nb; ++b) { const int32_t v = blk[b]; blk[b] = acc; acc += v; }
}
__global__ void k_scan_add(int32_t* a, long long len, const int32_t* blk) {
  const long long base = ((long long)blockIdx.x * NT + threadIdx.x) * SCAN_ITEMS;
  const int32_t off = blk[blockIdx.x];
  for (int u = 0; u < SCAN_ITEMS; ++u) {
    const long long i = base + u;
    if (i < len) a[i] += off;
  }
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

}  // namespace

struct plss_ctx {
  bool xdefer = false;         // K3 updates x every other step (K3_XDEFER; row-slab steps)
  int psi_dots = 0;            // row blocks: k_dots_tail leaves psi to K3 (K3_PSI)
  int dev = 0;
  cudaStream_t stream = nullptr;       // work stream (the caller's, or our own if it passed NULL)
  cudaStream_t user_stream = nullptr;  // the caller's stream
  bool own_stream = false;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  plss_matrix A{};
  Layout L{};
  int S = 1;
  int64_t m = 0, n = 0, nnz = 0;
  std::vector<int64_t> R, E;     // slab row bounds / entry bounds
  char* ws = nullptr;
  double *r = nullptr, *y = nullptr, *p = nullptr, *x = nullptr, *rec = nullptr;
  double* wi = nullptr;          // diagonal of WI (PLSS W), valid when `weighted`
  bool weighted = false;
  Ctl* ctl = nullptr;
  unsigned* counters = nullptr;
  double *part1 = nullptr, *part2 = nullptr, *part3 = nullptr, *partn = nullptr;
  double* scalars = nullptr;
  std::vector<SpmvSeg> seg1, seg2;
  std::vector<int> g1, g2;
  int g3 = 1, gdots = 1, gnorm = 1;
  int chunk = 16;
  cudaGraphExec_t graph_chunk = nullptr, graph_one = nullptr;
  // distributed (created by plss_create_dist, any nranks >= 1)
  bool dist = false;
  // the last K2 segment split into column chunks, each all-reduced on comm_stream while the next
  // chunk computes (drows: first row of each chunk and n + 1 at the end)
  std::vector<SpmvSeg> dch;
  std::vector<int> gch;
  std::vector<int64_t> drows;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_ch[DCH_MAX] = {}, ev_join = nullptr;
  // reduce-scatter / all-gather step (options.flags bit2): column shard [c0, c0 + nsh) of the
  // padded nranks x cnt vectors; scalars[4..7] = {rho, phi, psi, theta} partials, all-reduced
  bool rsag = false;
  int64_t cnt = 0, c0 = 0, nsh = 0;
  int rank = 0, nranks = 1;
  ncclComm_t comm = nullptr;
  // peer-memory all-reduce (options.flags bit3, peer_kernels.cuh): a region the library allocates
  // (cudaMalloc, so that CUDA IPC can map it) = [reduced y | rho][partial y | rho][flag block];
  // y points at the partial (what K1 / K2 write), yred at the reduced vector (what the dots, the
  // tails and K3 read); ptab holds every rank's region as mapped in this process
  // column blocks (plss_create_dist_cols): this rank owns columns [col_offset, col_offset + n) of
  // an m x n_global matrix; r (m) is replicated, x / p / y are this rank's column shards
  bool cols = false;
  int64_t col_offset = 0, n_global = 0;
  // row blocks (plss_create_dist): this rank owns rows [row_offset, row_offset + m) of m_global
  int64_t row_offset = 0, m_global = 0;
  // NCCL failure detection (dist_wait): the communicator was aborted after an asynchronous error
  // or a wait timeout; every later call on this ctx fails with PLSS_E_NCCL
  bool aborted = false;
  std::vector<void*> dbg_bufs;   // PLSS_DBG_CTA buffers
  std::vector<void*> chunk_bufs; // k_longchunks' chunk tables, row counters and partials (one per segment)
  char* slabmajor = nullptr;     // the slab-major CSC when SELL is on and a K2 segment still reads it
  cudaStream_t fork_stream = nullptr;          // k_longrows' concurrent stream (launch_spmv)
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  int fault_nccl = 0;            // PLSS_FAULT_NCCL=1 (tests): the first poll reports an error
  double wait_timeout_s = 600.0; // PLSS_WAIT_TIMEOUT_S
  bool peer = false;
  char* sym = nullptr;
  size_t sym_yb = 0;
  double* yred = nullptr;
  PeerTab ptab{};
  std::vector<void*> ipc_open;
  int peer_gx = 1;
  // solve state
  bool started = false;
  int maxit = 0, flags = 0;
  int32_t* h_done = nullptr;     // pinned [2]
  Ctl* h_ctl = nullptr;          // pinned staging
  cudaEvent_t ev[2] = {nullptr, nullptr};
  // randomized projection (plss_rp_*): shares r, p, x, ctl, rec and the K1 segments
  bool rp_started = false;
  RpArgs rp{};
  int rp_gspmm = 1, rp_gupd = 1;
  cudaGraphExec_t rp_graph_chunk = nullptr, rp_graph_one = nullptr;
  // PLSS Kaczmarz (plss_kz_*): shares r, p, x, ctl, rec and the K1 segments
  bool kz_started = false;
  KzArgs kz{};
  std::vector<SpmvSeg> kz_seg;   // K1 segments in plain mode: apk = A pk
  cudaGraphExec_t kz_graph_chunk = nullptr, kz_graph_one = nullptr;
  // growing-sketch engine (plss_eg_*): shares r, y, p, x, ctl, rec and the K1 / K2 segments
  bool eg_started = false;
  EgArgs eg{};
  std::vector<SpmvSeg> eg_seg;   // K2 segments gathering the sketch column: y = A^T s
  cudaGraphExec_t eg_graph_chunk = nullptr, eg_graph_one = nullptr;
  std::string err;
};

#define CK(call)                                                                    \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      set_err(ctx, std::string(#call) + ": " + cudaGetErrorString(e_));            \
      return PLSS_E_CUDA;                                                           \
    }                                                                               \
  } while (0)

#define NK(call)                                                                    \
  do {                                                                              \
    ncclResult_t e_ = (call);                                                       \
    if (e_ != ncclSuccess) {                                                        \
      set_err(ctx, std::string(#call) + ": " + ncclGetErrorString(e_));             \
      return PLSS_E_NCCL;                                                           \
    }                                                                               \
  } while (0)

static void set_err(plss_ctx* ctx, const std::string& s) {
  if (ctx) ctx->err = s;
  g_last_error = s;
}

// the long rows of a globally sorted segment: a warp per chunk (k_longchunks), else a CTA per row
template <int ROLE>
static void launch_long(const SpmvSeg& c, cudaStream_t st) {
  if (c.lchunk)
    k_longchunks<ROLE><<<(c.nchunks + NT / 32 - 1) / (NT / 32), NT, 0, st>>>(c);
  else
    k_longrows<ROLE><<<c.nlong, NT, 0, st>>>(c);
}

template <int ROLE>
static void launch_spmv(const SpmvSeg& a, int grid, cudaStream_t st) {
  if (a.fmt == 5)
    a.scb == 3 ? k_scalar<ROLE, 3><<<grid, NT, 0, st>>>(a) : k_scalar<ROLE, 2><<<grid, NT, 0, st>>>(a);
  else if (a.fmt == 2)
    k_sellw<ROLE><<<grid, NTW, (size_t)a.ring * 8, st>>>(a);
  else if (a.fmt == 3 && a.nlong > 0 && a.lin) {
    // gsort with long rows in chunks run by k_sell itself (phase 0): its long-row partial pair sits
    // after the CTAs' and arrives in the election as one more (never the last: its CTA is still out)
    SpmvSeg b = a;
    b.elect_extra = 1;
    b.elect_total = grid + 1;
    k_sell<ROLE, 1024, false, false, SIGMA, false, GS_SU, GS_NSB><<<grid, 1024, 0, st>>>(b);
  }
  else if (a.fmt == 3 && a.nlong > 0) {
    // gsort with long rows: the slices and k_longrows (one CTA per long row) run concurrently
    // (k_longrows forked onto a second stream, joined before the next launch): its CTAs fill the SMs
    // the slices' CTAs free. It publishes its dot terms in the partial slot after the slices' CTAs;
    // the slices' CTAs and its last CTA elect the finalizing CTA together
    SpmvSeg b = a;
    b.elect_extra = 1;
    SpmvSeg c = a;
    c.partial = a.partial + 2 * (size_t)grid;
    c.elect_total = grid + 1;
    cudaStream_t st2 = (cudaStream_t)a.fork_stream;
    if (st2) {
      cudaEventRecord((cudaEvent_t)a.fork_ev, st);
      cudaStreamWaitEvent(st2, (cudaEvent_t)a.fork_ev, 0);
      launch_long<ROLE>(c, st2);
      cudaEventRecord((cudaEvent_t)a.join_ev, st2);
      k_sell<ROLE, 1024, false, false, SIGMA, false, GS_SU, GS_NSB><<<grid, 1024, 0, st>>>(b);   // gsort: no y staging
      cudaStreamWaitEvent(st, (cudaEvent_t)a.join_ev, 0);
    } else {
      k_sell<ROLE, 1024, false, false, SIGMA, false, GS_SU, GS_NSB><<<grid, 1024, 0, st>>>(b);
      launch_long<ROLE>(c, st);
    }
  }
  else if (a.fmt == 3 && a.gsort)
    k_sell<ROLE, 1024, false, false, SIGMA, false, GS_SU, GS_NSB><<<grid, 1024, 0, st>>>(a);
  else if (a.fmt == 3 && ROLE >= ROLE_K2 && a.perm && !a.gsort && a.sig == SIGMA_WIDE)
    k_sell<ROLE, 1024, false, true, SIGMA_WIDE><<<grid, 1024, YSTAGE_SMEM_WIDE, st>>>(a);
  else if (a.fmt == 3 && ROLE >= ROLE_K2 && a.perm && !a.gsort)     // K2 with a sigma perm: staged y
    k_sell<ROLE, 1024, false, true><<<grid, 1024, YSTAGE_SMEM, st>>>(a);
  else if (a.fmt == 3 && a.stat == 2 && !a.perm)
    k_sell<ROLE, 1024, false, false, SIGMA, true, 6><<<grid, 1024, 0, st>>>(a);
  else if (a.fmt == 3 && a.stat && !a.perm)
    k_sell<ROLE, 1024, false, false, SIGMA, true><<<grid, 1024, 0, st>>>(a);
  else if (a.fmt == 3)
    k_sell<ROLE, 1024><<<grid, 1024, 0, st>>>(a);
  else if (a.fmt == 1)
    k_sell<ROLE><<<grid, NT, 0, st>>>(a);
  else
    k_spmv<ROLE><<<grid, NTS, Stage<ROLE>::SMEM, st>>>(a);
}

// order our work stream after / before the caller's stream when they differ
static plss_status sync_in(plss_ctx* ctx) {
  if (!ctx->own_stream) return PLSS_OK;
  CK(cudaEventRecord(ctx->ev_in, ctx->user_stream));
  CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_in, 0));
  return PLSS_OK;
}
static plss_status sync_out(plss_ctx* ctx) {
  if (!ctx->own_stream) return PLSS_OK;
  CK(cudaEventRecord(ctx->ev_out, ctx->stream));
  CK(cudaStreamWaitEvent(ctx->user_stream, ctx->ev_out, 0));
  return PLSS_OK;
}

static int grid_for(int64_t work_units, int occ_per_sm, int sms) {
  int64_t g = std::min<int64_t>(work_units, (int64_t)occ_per_sm * sms);
  g = std::min<int64_t>(g, MAXG);
  return (int)std::max<int64_t>(1, g);
}

// peer-memory reduce of chunk c = elements [lo, hi) of y | rho (this rank's shard, to every rank)
static void peer_reduce(plss_ctx* ctx, int c, int64_t lo, int64_t hi, cudaStream_t s) {
  k_peer_reduce<<<dim3(ctx->peer_gx, 1), PEER_NT, 0, s>>>(ctx->ptab, ctx->nranks, ctx->rank, c, (long long)lo,
                                                          (long long)hi, ctx->ctl);
}
static int peer_nch(const plss_ctx* ctx) { return ctx->dch.empty() ? 1 : (int)ctx->dch.size(); }
// all chunks, in order, on one stream (unchunked step, plss_profile)
static void peer_reduce_all(plss_ctx* ctx, cudaStream_t s) {
  if (ctx->dch.empty()) {
    peer_reduce(ctx, 0, 0, ctx->n + 1, s);
  } else {
    for (int c = 0; c < (int)ctx->dch.size(); ++c) peer_reduce(ctx, c, ctx->drows[c], ctx->drows[c + 1], s);
  }
}

// column-block step: K1 (u <- u - A_g p_g; u = r on rank 0, 0 elsewhere), all-reduce of u | theta_g,
// rho tail, K2 (y_g = A_g^T r), phi / psi partials, all-reduce of 2 scalars, y tail, K3 on the
// shard (theta_g into r[m] for the next all-reduce), ranks > 0 zero u again
static plss_status enqueue_step_cols(plss_ctx* ctx) {
  cudaStream_t st = ctx->stream;
  const int64_t m = ctx->m;
  double* sc = ctx->scalars + 4;
  for (int s = 0; s < ctx->S; ++s) launch_spmv<ROLE_K1>(ctx->seg1[s], ctx->g1[s], st);
  NK(ncclAllReduce(ctx->r, ctx->r, (size_t)m + 1, ncclFloat64, ncclSum, ctx->comm, st));
  k_rho_tail<<<ctx->gnorm, NT, 0, st>>>(ctx->r, m, ctx->ctl, ctx->rec, ctx->partn, ctx->counters + 3);
  for (int s = 0; s < ctx->S; ++s) launch_spmv<ROLE_K2>(ctx->seg2[s], ctx->g2[s], st);
  k_dots_shard<<<ctx->gdots, NT, 0, st>>>(ctx->y, ctx->p, ctx->n, ctx->ctl, ctx->part2, ctx->counters + 1,
                                          ctx->wi, sc);
  NK(ncclAllReduce(sc + 1, sc + 1, 2, ncclFloat64, ncclSum, ctx->comm, st));
  k_tail_phi<<<1, 1, 0, st>>>(ctx->ctl, ctx->rec, sc);
  k_pxupdate<<<ctx->g3, NT, 0, st>>>(ctx->p, ctx->y, ctx->x, ctx->n, ctx->ctl, ctx->rec, ctx->part3,
                                     ctx->counters + 2, ctx->wi, ctx->r + m);
  if (ctx->rank > 0 && m > 0) CK(cudaMemsetAsync(ctx->r, 0, 8 * (size_t)m, st));
  CK(cudaGetLastError());
  return PLSS_OK;
}

// enqueue one loop step (also used inside graph capture)
// K3's options on the row-slab steps (one device, or row blocks with the all-reduce / peer step): psi
// summed in K3 when K2's finalizing segment (or k_dots_tail) left it (R25), x updated every
// other step (K3_XDEFER, flushed by plss_finish)
static int k3_opts(const plss_ctx* ctx) {
  if (ctx->cols || ctx->rsag) return 0;
  const bool psi = ctx->dist ? ctx->psi_dots : ctx->seg2[ctx->S - 1].psi3;
  return (psi ? K3_PSI : 0) | (ctx->xdefer ? K3_XDEFER : 0);
}

static plss_status enqueue_step(plss_ctx* ctx) {
  if (ctx->cols) return enqueue_step_cols(ctx);
  cudaStream_t st = ctx->stream;
  const bool chunked = ctx->dist && !ctx->dch.empty();
  for (int s = 0; s < ctx->S; ++s) {
    launch_spmv<ROLE_K1>(ctx->seg1[s], ctx->g1[s], st);
    if (chunked && s == ctx->S - 1) {
      // last slab: column chunks, each all-reduced on comm_stream while the next one computes
      for (size_t c = 0; c < ctx->dch.size(); ++c) {
        launch_spmv<ROLE_K2>(ctx->dch[c], ctx->gch[c], st);
        CK(cudaEventRecord(ctx->ev_ch[c], st));
        CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_ch[c], 0));
        if (ctx->peer)
          peer_reduce(ctx, (int)c, ctx->drows[c], ctx->drows[c + 1], ctx->comm_stream);
        else
          NK(ncclAllReduce(ctx->y + ctx->drows[c], ctx->y + ctx->drows[c], (size_t)(ctx->drows[c + 1] - ctx->drows[c]),
                           ncclFloat64, ncclSum, ctx->comm, ctx->comm_stream));
      }
      CK(cudaEventRecord(ctx->ev_join, ctx->comm_stream));
      CK(cudaStreamWaitEvent(st, ctx->ev_join, 0));
    } else if (ctx->seg2[s].finalize) {
      launch_spmv<ROLE_K2DOTS>(ctx->seg2[s], ctx->g2[s], st);
    } else {
      launch_spmv<ROLE_K2>(ctx->seg2[s], ctx->g2[s], st);
    }
  }
  if (ctx->rsag) {
    // reduce-scatter y to this rank's shard, shard dots, one all-reduce of 4 scalars, the tails,
    // K3 on the shard, all-gather p (K1 gathers all of p)
    double* sc = ctx->scalars + 4;
    NK(ncclReduceScatter(ctx->y, ctx->y + ctx->c0, (size_t)ctx->cnt, ncclFloat64, ncclSum, ctx->comm, st));
    k_dots_shard<<<ctx->gdots, NT, 0, st>>>(ctx->y + ctx->c0, ctx->p + ctx->c0, ctx->nsh, ctx->ctl, ctx->part2,
                                            ctx->counters + 1, ctx->wi ? ctx->wi + ctx->c0 : nullptr, sc);
    NK(ncclAllReduce(sc, sc, 4, ncclFloat64, ncclSum, ctx->comm, st));
    k_tail_rsag<<<1, 1, 0, st>>>(ctx->ctl, ctx->rec, sc);
    k_pxupdate<<<ctx->g3, NT, 0, st>>>(ctx->p + ctx->c0, ctx->y + ctx->c0, ctx->x + ctx->c0, ctx->nsh, ctx->ctl, ctx->rec,
                                       ctx->part3, ctx->counters + 2, ctx->wi ? ctx->wi + ctx->c0 : nullptr, sc + 3);
    NK(ncclAllGather(ctx->p + ctx->c0, ctx->p, (size_t)ctx->cnt, ncclFloat64, ctx->comm, st));
    CK(cudaGetLastError());
    return PLSS_OK;
  }
  double* yv = ctx->y;
  if (ctx->dist) {
    if (ctx->peer) {
      if (!chunked) peer_reduce(ctx, 0, 0, ctx->n + 1, st);
      k_peer_wait<<<1, 64, 0, st>>>(ctx->ptab, ctx->nranks, peer_nch(ctx), ctx->rank, ctx->ctl);
      yv = ctx->yred;
    } else if (!chunked) {
      NK(ncclAllReduce(ctx->y, ctx->y, (size_t)ctx->n + 1, ncclFloat64, ncclSum, ctx->comm, st));
    }
    k_dots_tail<<<ctx->gdots, NT, 0, st>>>(yv, ctx->p, ctx->n, yv + ctx->n, ctx->ctl, ctx->rec,
                                           ctx->part2, ctx->counters + 1, ctx->wi, ctx->psi_dots);
  }
  k_pxupdate<<<ctx->g3, NT, 0, st>>>(ctx->p, yv, ctx->x, ctx->n, ctx->ctl, ctx->rec, ctx->part3,
                                     ctx->counters + 2, ctx->wi, nullptr, k3_opts(ctx));
  CK(cudaGetLastError());
  return PLSS_OK;
}

static plss_status build_graph(plss_ctx* ctx, int iters, cudaGraphExec_t* out) {
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  plss_status st = PLSS_OK;
  for (int i = 0; i < iters && st == PLSS_OK; ++i) st = enqueue_step(ctx);
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
  if (st != PLSS_OK) return st;
  CK(e);
  CK(cudaGraphInstantiate(out, g, 0));
  CK(cudaGraphDestroy(g));
  return PLSS_OK;
}

static plss_status scan_excl(plss_ctx* ctx, int32_t* a, long long len, int32_t* blk) {
  const unsigned nblk = (unsigned)((len + NT * SCAN_ITEMS - 1) / (NT * SCAN_ITEMS));
  k_scan_local<<<nblk, NT, 0, ctx->stream>>>(a, len, blk);
  k_scan_blocks<<<1, 1, 0, ctx->stream>>>(blk, (int)nblk);
  k_scan_add<<<nblk, NT, 0, ctx->stream>>>(a, len, blk);
  CK(cudaGetLastError());
  return PLSS_OK;
}

// tiles of one segment: descriptors desc[0..nt] (desc[nt] = {nrows, ptr[nrows]})
static plss_status build_tiles(plss_ctx* ctx, const int32_t* ptr, int64_t nrows, int64_t e0, int2* desc,
                               int64_t cap, int64_t* nt_out) {
  cudaStream_t st = ctx->stream;
  int32_t* flag = (int32_t*)(ctx->ws + ctx->L.scratch);
  int32_t* blk = (int32_t*)(ctx->ws + ctx->L.scratch_blk);
  const long long len = nrows + 1;
  const unsigned g = (unsigned)((len + 255) / 256);
  k_tile_mark<<<g, 256, 0, st>>>(ptr, nrows, e0, flag);
  if (scan_excl(ctx, flag, len, blk) != PLSS_OK) return PLSS_E_CUDA;
  int32_t nt = 0;
  CK(cudaMemcpyAsync(&nt, flag + nrows, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (nt + 1 > cap) { set_err(ctx, "tile descriptor bound exceeded"); return PLSS_E_CUDA; }
  k_tile_desc<<<g, 256, 0, st>>>(ptr, nrows, e0, flag, desc);
  CK(cudaGetLastError());
  *nt_out = nt;
  return PLSS_OK;
}

template <int ROLE>
static cudaError_t smem_attr(int* occ) {
  cudaError_t e = cudaFuncSetAttribute(k_spmv<ROLE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Stage<ROLE>::SMEM);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, k_spmv<ROLE>, NTS, Stage<ROLE>::SMEM);
  *occ = std::max(1, *occ);
  return e;
}

static plss_status set_smem_attrs(plss_ctx* ctx, int occ[4]) {
  CK(smem_attr<ROLE_PLAIN>(&occ[ROLE_PLAIN]));
  CK(smem_attr<ROLE_K1>(&occ[ROLE_K1]));
  CK(smem_attr<ROLE_K2>(&occ[ROLE_K2]));
  CK(smem_attr<ROLE_K2DOTS>(&occ[ROLE_K2DOTS]));
  return PLSS_OK;
}


// SELL pool cursor of one side (K1 or K2)
struct SellPool {
  int32_t *idx, *perm, *sptr;
  double* val;
  int64_t cap, slots, sp;      // capacities
  int64_t used, used_slots, used_sp;
  int2* win;                   // window descriptors (one per NSB-slice block)
  int64_t wcap, used_w;
  int32_t* cblk;               // CTA block ranges (MAXG+1 per segment)
  int64_t used_c;
  int32_t* aux;                // long-row lists and unit-weight prefixes (global-sort segments)
  int64_t auxn, used_aux;
};

static int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return (e && *e) ? std::atoi(e) : dflt;
}

// Give a SELL segment a shared-memory window of its gathered vector g (length glen) when enough of
// its entries fall into per-block windows of `win` doubles ("Windows").
// One 1024-thread CTA per SM over contiguous entry-balanced slice ranges (fmt 3).
static plss_status make_contig(plss_ctx* ctx, SpmvSeg& a, SellPool& pool, int sms, int* grid_out) {
  if (a.fmt != 1) return PLSS_OK;
  const int nunits = a.nslices;                      // long rows run in k_longrows (launch_spmv)
  const int NSB = a.gsort ? GS_NSB : nsb_of(a.sig ? a.sig : SIGMA);   // the k_sell instantiation's block
  const int nblocks = (nunits + NSB - 1) / NSB;
  // a gsort segment's long rows run concurrently in k_longrows (launch_spmv): leave them SMs in
  // proportion to their share of the entries (PLSS_LSHARE percent of it)
  int sms_k = sms;
  if (a.gsort && a.nlong > 0 && a.long_entries > 0) {
    const double frac = (double)a.long_entries / (double)(a.long_entries + a.short_entries);
    sms_k = std::max(1, sms - (int)std::lround(sms * frac * env_int("PLSS_LSHARE", 0) / 100.0));
  }
  const int grid = std::max(1, std::min(std::min(nblocks, sms_k * (a.gsort ? GS_MINB : 1)), MAXG));
  int32_t* cblk = pool.cblk + pool.used_c;
  // CTA balance: a unit costs its stored entries plus a fixed overhead (metadata loads, row
  // outputs, dot partial); sigma-permuted slices also pay the scattered / staged y. Measured best:
  // 256 for sigma-permuted ones (C5 K2 +3%), 48 for globally sorted ones at single-slice
  // granularity (GS_NSB; 32 with blocks of 16: C4's K1 0.160 -> 0.123 ms when the CTAs of long
  // rows were the stragglers, scripts/cta_balance.py; 48 vs 32 since k_longchunks: C4 0.2303 ->
  // 0.2274, C4-alt 0.3910 -> 0.3834 ms per step), 128 otherwise.
  const int uc = (a.perm && !a.gsort) ? env_int("PLSS_UC_SIG", 256)
                 : a.gsort ? env_int("PLSS_UC_GS", 48) : env_int("PLSS_UC", 128);
  // one-step slices in k_sell's batched phase 2 (globally sorted): PLSS_UC_S1 per slice beyond its
  // 32 stored entries
  if (a.uw && a.s1on)
    k_cta_ranges<<<(grid + 256) / 256, 256, 0, ctx->stream>>>(a.uw, 1, nunits, NSB, nblocks, grid, cblk, uc,
                                                              a.s1beg, env_int("PLSS_UC_S1", 16));
  else if (a.uw)
    k_cta_ranges<<<(grid + 256) / 256, 256, 0, ctx->stream>>>(a.uw, 1, nunits, NSB, nblocks, grid, cblk, uc);
  else
    k_cta_ranges<<<(grid + 256) / 256, 256, 0, ctx->stream>>>(a.sptr, 32, nunits, NSB, nblocks, grid, cblk, uc);
  CK(cudaGetLastError());
  pool.used_c += MAXG + 1;
  a.cblk = cblk;
  a.slpart = (double*)(ctx->ws + ctx->L.slpart);
  a.fmt = 3;
  *grid_out = grid;
  return PLSS_OK;
}

// Split a fmt 3 K2 segment with a sigma perm into `nch` column chunks at sigma-window boundaries:
// slices [sl0, sl1) of window-aligned ranges keep their absolute rows (perm) and y-staging windows
// (wrow0), and get their own entry-balanced CTA ranges. Used by the distributed step to all-reduce
// a finished chunk of y while the next one computes.
static plss_status make_chunks(plss_ctx* ctx, const SpmvSeg& a, SellPool& pool, int sms, int nch) {
  ctx->dch.clear();
  ctx->gch.clear();
  ctx->drows.clear();
  if (a.fmt != 3 || !a.perm || a.gsort || nch < 2) return PLSS_OK;
  const int sigw = a.sig ? a.sig : SIGMA, SPW = sigw / 32;
  const int nwin = (a.nslices + SPW - 1) / SPW;
  nch = std::min(nch, std::min(nwin, DCH_MAX));
  if (nch < 2) return PLSS_OK;
  for (int c = 0; c < nch; ++c) {
    const int w0 = (int)((int64_t)nwin * c / nch), w1 = (int)((int64_t)nwin * (c + 1) / nch);
    SpmvSeg b = a;
    const int sl0 = w0 * SPW, sl1 = std::min(w1 * SPW, a.nslices);
    b.sptr = a.sptr + sl0;
    b.perm = a.perm + (size_t)sl0 * 32;
    b.nslices = sl1 - sl0;
    b.wrow0 = w0 * sigw;
    b.fmt = 1;                                       // make_contig turns it into fmt 3 with its ranges
    b.uw = nullptr;
    int grid = 1;
    plss_status st = make_contig(ctx, b, pool, sms, &grid);
    if (st != PLSS_OK) return st;
    ctx->dch.push_back(b);
    ctx->gch.push_back(grid);
    ctx->drows.push_back((int64_t)w0 * sigw);
  }
  ctx->drows.push_back(ctx->n + 1);                  // the last chunk's all-reduce carries rho too
  CK(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
  for (int c = 0; c < nch; ++c) CK(cudaEventCreateWithFlags(&ctx->ev_ch[c], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
  return PLSS_OK;
}

static plss_status try_window(plss_ctx* ctx, SpmvSeg& a, const double* g, int64_t glen, int64_t nnz_seg,
                              int win, int nsb, SellPool& pool, int sms, int* grid_out) {
  cudaStream_t st = ctx->stream;
  if (a.fmt != 1 || a.gsort || win <= 0 || nnz_seg == 0) return PLSS_OK;
  win &= ~7;
  if (glen - 2 < win) win = (int)((glen - 2) & ~7ll);
  if (win < 256) return PLSS_OK;
  nsb = std::max(4, std::min(nsb, 64));
  const int ring = win + win / 2 + 8;              // advance allowance: (WST-1) blocks in flight
  if ((size_t)ring * 8 > 200 * 1024) return PLSS_OK;
  const int nblocks = (a.nslices + nsb - 1) / nsb;
  if (pool.used_w + nblocks > pool.wcap) return PLSS_OK;
  int2* wlo = pool.win + pool.used_w;
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sellw<ROLE_K2DOTS>, NTW, (size_t)ring * 8));
  if (occ < 1) return PLSS_OK;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(nblocks, (int64_t)occ * sms), MAXG));
  // bins: win/4 wide (at most 16384 of them), windows of kb bins
  int64_t bw = std::max<int64_t>(win / 4, (glen + 16383) / 16384);
  const int nbins = (int)((glen + bw - 1) / bw);
  const int kb = (int)std::max<int64_t>(1, win / bw);
  const int goff = (int)((reinterpret_cast<uintptr_t>(g) >> 3) & 1);
  unsigned long long* covered = (unsigned long long*)(ctx->ws + ctx->L.err + 16);
  CK(cudaMemsetAsync(covered, 0, 8, st));
  k_win_choose<<<nblocks, 256, (size_t)nbins * 4, st>>>(a.sptr, a.idx, a.nslices, nsb, (int)glen, win, (int)bw,
                                                         nbins, kb, goff, std::max(64, win / 16), wlo, covered);
  CK(cudaGetLastError());
  unsigned long long cov = 0;
  CK(cudaMemcpyAsync(&cov, covered, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if ((double)cov < 0.1 * (double)nnz_seg) return PLSS_OK;          // too little locality
  int32_t* cblk = pool.cblk + pool.used_c;
  k_cta_ranges<<<(grid + 256) / 256, 256, 0, st>>>(a.sptr, 32, a.nslices, nsb, nblocks, grid, cblk, 128);
  k_win_chain<<<(grid + 255) / 256, 256, 0, st>>>(wlo, cblk, grid, win, ring);
  CK(cudaGetLastError());
  a.cblk = cblk;
  a.slpart = (double*)(ctx->ws + ctx->L.slpart);
  pool.used_c += MAXG + 1;
  a.fmt = 2;
  a.win = win;
  a.ring = ring;
  a.nblocks = nblocks;
  a.glen = (int32_t)glen;
  a.nsb = nsb;
  a.wlo = wlo;
  pool.used_w += nblocks;
  *grid_out = grid;
  return PLSS_OK;
}

// Convert one segment (CSR-like: ptr[nrows+1] absolute positions, idx, val) to SELL-32 if the
// padding stays small: unsorted when rows are (nearly) uniform, else sigma-sorted windows of 256.
// Rows too irregular for windowed sigma sorting (power-law lengths): sort ALL rows of the segment
// by length (setup only, on the host: a stable counting sort), put rows of <= LONGROW entries into
// SELL-32 slices (padding from equal-length neighbours only) and make every longer row a warp unit
// (fmt 3 only; its sum is a fixed lane-strided tree, like the CSR-tile kernel's long rows).
static plss_status try_sell_global(plss_ctx* ctx, SpmvSeg& a, int64_t nnz_seg, SellPool& pool) {
  cudaStream_t st = ctx->stream;
  const int64_t nrows = a.nrows;
  if (!env_int("PLSS_GSORT", 1)) return PLSS_OK;
  std::vector<int32_t> len(nrows);
  CK(cudaMemcpyAsync(len.data(), ctx->ws + ctx->L.scratch, 4 * (size_t)nrows, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::vector<int64_t> cnt(LONGROW + 2, 0);
  std::vector<int32_t> lrows;
  for (int64_t i = 0; i < nrows; ++i) {
    if (len[i] > LONGROW) lrows.push_back((int32_t)i); else cnt[len[i]]++;
  }
  const int64_t nshort = nrows - (int64_t)lrows.size();
  const int64_t nsl = (nshort + 31) / 32;
  const int64_t nlr = (int64_t)lrows.size();
  const int64_t nunits = nsl;                       // long rows run in k_longrows, not as k_sell units
  const int64_t aux_need = 3 * nlr + 4 * nlr + 2 + nunits + 1;   // lrows, lbeg (2), lrowd (2 doubles), align, uw
  if (pool.used_slots + nsl * 32 > pool.slots || pool.used_sp + nsl + 1 > pool.sp ||
      pool.used_aux + aux_need > pool.auxn)
    return PLSS_OK;
  // stable counting sort, length descending
  std::vector<int64_t> off(LONGROW + 2, 0);
  for (int l = LONGROW, acc = 0; l >= 0; --l) { off[l] = acc; acc += (int)cnt[l]; }
  std::vector<int32_t> perm(nsl * 32, -1);
  for (int64_t i = 0; i < nrows; ++i)
    if (len[i] <= LONGROW) perm[off[len[i]]++] = (int32_t)i;
  std::vector<int32_t> sp(nsl + 1, 0), uw(nunits + 1, 0);
  int64_t steps = 0, stored = 0;
  for (int64_t s2 = 0; s2 < nsl; ++s2) {
    sp[s2] = (int32_t)steps;
    uw[s2] = (int32_t)stored;
    const int32_t r = perm[s2 * 32];
    const int64_t L = r >= 0 ? len[r] : 0;          // longest row of the slice (sorted)
    steps += L;
    stored += 32 * L;
  }
  sp[nsl] = (int32_t)steps;
  uw[nunits] = (int32_t)stored;
  // the tail of one-step slices, then of empty ones (sorted last): k_sell's batched phase 2
  int64_t s1beg = nsl, s1end = nsl;
  for (int64_t s2 = nsl; s2 > 0 && sp[s2] - sp[s2 - 1] <= 1; --s2) s1beg = s2 - 1;
  for (int64_t s2 = nsl; s2 > s1beg && sp[s2] == sp[s2 - 1]; --s2) s1end = s2 - 1;
  a.short_entries = stored;
  for (size_t k = 0; k < lrows.size(); ++k) stored += len[lrows[k]];
  a.long_entries = stored - a.short_entries;
  if (stored >= (1ll << 31) || pool.used + steps * 32 > pool.cap) return PLSS_OK;
  if ((double)(steps * 32) > 1.15 * (double)nnz_seg + 32.0 * 32 * (LONGROW + 1)) return PLSS_OK;
  int32_t* d_perm = pool.perm + pool.used_slots;
  int32_t* d_sp = pool.sptr + pool.used_sp;
  // long rows longest first (CTA k of k_longrows takes the k-th: the longest start in the first
  // wave), each with its absolute entry range (no lrows -> row pointer load chain on the device)
  int32_t p0 = 0;
  CK(cudaMemcpyAsync(&p0, a.ptr, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::vector<int64_t> rstart;
  if (!lrows.empty()) {
    std::vector<int64_t> pre(nrows + 1, p0);
    for (int64_t i = 0; i < nrows; ++i) pre[i + 1] = pre[i] + len[i];
    std::stable_sort(lrows.begin(), lrows.end(), [&](int32_t x, int32_t y) { return len[x] > len[y]; });
    rstart.resize(lrows.size());
    for (size_t k = 0; k < lrows.size(); ++k) rstart[k] = pre[lrows[k]];
  }
  std::vector<int32_t> lbeg(2 * lrows.size());
  for (size_t k = 0; k < lrows.size(); ++k) {
    lbeg[2 * k] = (int32_t)rstart[k];
    lbeg[2 * k + 1] = (int32_t)(rstart[k] + len[lrows[k]]);
  }
  int32_t* d_lrows = pool.aux + pool.used_aux;
  int32_t* d_lbeg = d_lrows + nlr;
  double* d_lrowd = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(d_lbeg + 2 * nlr) + 7) & ~(uintptr_t)7);
  int32_t* d_uw = reinterpret_cast<int32_t*>(d_lrowd + 2 * nlr);
  CK(cudaMemcpyAsync(d_perm, perm.data(), 4 * perm.size(), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_sp, sp.data(), 4 * sp.size(), cudaMemcpyHostToDevice, st));
  if (!lrows.empty()) {
    CK(cudaMemcpyAsync(d_lrows, lrows.data(), 4 * lrows.size(), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_lbeg, lbeg.data(), 4 * lbeg.size(), cudaMemcpyHostToDevice, st));
  }
  CK(cudaMemcpyAsync(d_uw, uw.data(), 4 * uw.size(), cudaMemcpyHostToDevice, st));
  // k_longchunks: the long rows in chunks of LCH entries (longest row first, a row's chunks
  // consecutive), per row its chunk count and a finished-chunk counter, per chunk a partial
  std::vector<int32_t> lnch(lrows.size());
  std::vector<int4> chunks;
  if (!lrows.empty() && env_int("PLSS_LCHUNK", 1)) {
    for (size_t k = 0; k < lrows.size(); ++k) {
      const int32_t first = (int32_t)chunks.size();
      for (int32_t e = lbeg[2 * k]; e < lbeg[2 * k + 1]; e += LCH)
        chunks.push_back(make_int4(e, std::min(e + LCH, lbeg[2 * k + 1]), (int32_t)k, first));
      lnch[k] = (int32_t)chunks.size() - first;
    }
    const size_t ngroup = (lnch.size() + 31) / 32;
    const size_t b_ch = align_up(16 * chunks.size()), b_n = align_up(4 * lnch.size()), b_c = align_up(4 * lnch.size()),
                 b_gc = align_up(4 * ngroup), b_gd = align_up(16 * ngroup);
    char* buf = nullptr;
    CK(cudaMalloc((void**)&buf, b_ch + b_n + b_c + b_gc + b_gd + 8 * chunks.size()));
    ctx->chunk_bufs.push_back(buf);
    CK(cudaMemcpyAsync(buf, chunks.data(), 16 * chunks.size(), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(buf + b_ch, lnch.data(), 4 * lnch.size(), cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(buf + b_ch + b_n, 0, b_c + b_gc, st));     // row and group counters
    a.lchunk = (const int4*)buf;
    a.lnch = (const int32_t*)(buf + b_ch);
    a.lrcnt = (unsigned*)(buf + b_ch + b_n);
    a.lgcnt = (unsigned*)(buf + b_ch + b_n + b_c);
    a.lgd = (double*)(buf + b_ch + b_n + b_c + b_gc);
    a.lcpart = (double*)(buf + b_ch + b_n + b_c + b_gc + b_gd);
    a.nchunks = (int32_t)chunks.size();
    a.lin = env_int("PLSS_LIN", 0);                 // opt-in: measured slower
  }
  int32_t* sidx = pool.idx + pool.used;
  double* sval = pool.val + pool.used;
  if (nsl > 0)
    k_sell_fill<<<(unsigned)((nsl * 32 + 255) / 256), 256, 0, st>>>(a.ptr, a.idx, a.val, d_perm, nrows, nsl, d_sp,
                                                                    sidx, sval);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));                    // the host vectors go out of scope
  a.fmt = 1;
  a.gsort = 1;
  a.nslices = (int32_t)nsl;
  a.sptr = d_sp;
  a.perm = d_perm;
  a.nlong = (int32_t)lrows.size();
  a.lrows = d_lrows;
  a.lrowd = d_lrowd;
  a.lbeg = d_lbeg;
  a.lcounter = ctx->counters + 8;
  a.lptr = a.ptr;
  a.lidx = a.idx;
  a.lval = a.val;
  a.uw = d_uw;
  a.idx = sidx;
  a.val = sval;
  a.s1on = s1beg < nsl && env_int("PLSS_S1", 1);
  a.s1beg = (int32_t)s1beg;
  a.s1end = (int32_t)s1end;
  a.s1step0 = sp[s1beg];
  pool.used += steps * 32;
  pool.used_slots += nsl * 32;
  pool.used_sp += nsl + 1;
  pool.used_aux += aux_need;
  return PLSS_OK;
}

// A segment of short rows (mean <= SCALAR_MEAN entries, none above SCALAR_MAX: C4's and C4-alt's
// columns) takes fmt 5, a thread per row over its own arrays (k_scalar); PLSS_SCALAR=0 disables.
static plss_status try_scalar(plss_ctx* ctx, SpmvSeg& a, int64_t nnz_seg, int sms, int* grid_out) {
  if (!env_int("PLSS_SCALAR", 1) || a.nrows == 0 || nnz_seg > (int64_t)SCALAR_MEAN * a.nrows) return PLSS_OK;
  cudaStream_t st = ctx->stream;
  int* d_max = (int*)(ctx->ws + ctx->L.err + 8);
  CK(cudaMemsetAsync(d_max, 0, 4, st));
  k_max_len<<<(unsigned)((a.nrows + 255) / 256), 256, 0, st>>>(a.ptr, a.nrows, d_max);
  CK(cudaGetLastError());
  int mx = 0;
  CK(cudaMemcpyAsync(&mx, d_max, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (mx > SCALAR_MAX) return PLSS_OK;
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_scalar<ROLE_K2DOTS>, NT, 0));
  a.fmt = 5;
  a.scb = (nnz_seg < 2 * a.nrows && env_int("PLSS_SCB3", 1)) ? 3 : 2;   // mean < 2 entries: 3 in flight
  *grid_out = (int)std::max<int64_t>(1, std::min<int64_t>((a.nrows + NT - 1) / NT, (int64_t)std::max(1, occ) * sms));
  *grid_out = std::min(*grid_out, MAXG);
  return PLSS_OK;
}

static plss_status try_sell(plss_ctx* ctx, SpmvSeg& a, int64_t nnz_seg, SellPool& pool, int sms, int occ,
                            bool wide_ok = false) {
  cudaStream_t st = ctx->stream;
  const int64_t nrows = a.nrows;
  const int64_t nsl = (nrows + 31) / 32;
  if (nrows == 0 || nnz_seg == 0) return PLSS_OK;
  if (pool.used_slots + nsl * 32 > pool.slots || pool.used_sp + nsl + 1 > pool.sp) return PLSS_OK;
  int32_t* len = (int32_t*)(ctx->ws + ctx->L.scratch);
  int32_t* blk = (int32_t*)(ctx->ws + ctx->L.scratch_blk);
  int32_t* sp = pool.sptr + pool.used_sp;
  int32_t* perm = pool.perm + pool.used_slots;
  const unsigned g = (unsigned)((nrows + 255) / 256);
  const unsigned gs = (unsigned)((nsl + 1 + 255) / 256);
  k_row_len<<<g, 256, 0, st>>>(a.ptr, nrows, len);
  int64_t steps = 0;
  const int32_t* use_perm = nullptr;
  // pass 0: no sort; 1: sigma windows of SIGMA rows; 2 (K2 segments): of SIGMA_WIDE rows (sparse
  // columns of power-law matrices: C4 0.335 vs 0.355 ms per step)
  const int npass = wide_ok ? 3 : 2;
  a.sig = 0;
  for (int pass = 0; pass < npass; ++pass) {
    if (pass == 1) {
      k_sigma_sort<SIGMA><<<(unsigned)((nrows + SIGMA - 1) / SIGMA), SIGMA_NT, 0, st>>>(len, nrows, nsl * 32, perm);
      use_perm = perm;
    } else if (pass == 2) {
      k_sigma_sort<SIGMA_WIDE><<<(unsigned)((nrows + SIGMA_WIDE - 1) / SIGMA_WIDE), SIGMA_NT, 0, st>>>(len, nrows,
                                                                                                   nsl * 32, perm);
      a.sig = SIGMA_WIDE;
    }
    k_slice_len<<<gs, 256, 0, st>>>(len, use_perm, nrows, nsl, sp);
    if (scan_excl(ctx, sp, nsl + 1, blk) != PLSS_OK) return PLSS_E_CUDA;
    int32_t tot[2] = {0, 0};                          // sp[nsl-1], sp[nsl]
    CK(cudaMemcpyAsync(tot, sp + nsl - 1, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    steps = tot[1];
    // padding of the partial last slice is bounded (one slice per segment): not counted
    const int64_t padded = steps * 32 - (nsl * 32 - nrows) * (int64_t)(tot[1] - tot[0]);
    const double limit = pass == 0 ? 1.03 : 1.15;
    if ((double)padded <= limit * (double)nnz_seg + 1024.0) break;
    if (pass == npass - 1) { a.sig = 0; return try_sell_global(ctx, a, nnz_seg, pool); }   // power-law rows
  }
  if (pool.used + steps * 32 > pool.cap) return PLSS_OK;
  int32_t* sidx = pool.idx + pool.used;
  double* sval = pool.val + pool.used;
  k_sell_fill<<<(unsigned)((nsl * 32 + 255) / 256), 256, 0, st>>>(a.ptr, a.idx, a.val, use_perm, nrows, nsl, sp,
                                                                  sidx, sval);
  CK(cudaGetLastError());
  a.fmt = 1;
  a.nslices = (int32_t)nsl;
  a.sptr = sp;
  a.perm = use_perm;
  a.idx = sidx;
  a.val = sval;
  pool.used += steps * 32;
  pool.used_slots += nsl * 32;
  pool.used_sp += nsl + 1;
  (void)sms; (void)occ;
  return PLSS_OK;
}

static plss_status setup(plss_ctx* ctx, const plss_matrix* A, const plss_options* opt, void* workspace,
                         size_t ws_bytes, void* stream, bool dist) {
  ctx->A = *A;
  ctx->m = A->m; ctx->n = A->n; ctx->nnz = A->nnz;
  if (!compute_layout(A, opt, dist, &ctx->L)) { set_err(ctx, "invalid matrix sizes"); return PLSS_E_DIM; }
  if (!workspace || ws_bytes < ctx->L.total) { set_err(ctx, "workspace too small"); return PLSS_E_DIM; }
  if ((reinterpret_cast<uintptr_t>(workspace) & (ALIGN - 1)) != 0) { set_err(ctx, "workspace not 256-byte aligned"); return PLSS_E_INVALID; }
  if (!A->row_ptr || !A->col_ptr || (A->nnz > 0 && (!A->col_idx || !A->val || !A->row_idx || !A->val_t))) {
    set_err(ctx, "NULL matrix array"); return PLSS_E_INVALID;
  }
  if (opt && (opt->flags & ~15) != 0) { set_err(ctx, "unknown options.flags bits"); return PLSS_E_INVALID; }
  if (opt && (opt->flags & 8)) {
    if (!dist) { set_err(ctx, "options.flags bit3 needs a distributed ctx"); return PLSS_E_INVALID; }
    if (opt->flags & 4) { set_err(ctx, "options.flags bit2 and bit3 are exclusive"); return PLSS_E_INVALID; }
    if (ctx->nranks > PEER_MAX) { set_err(ctx, "peer-memory step: at most 8 ranks"); return PLSS_E_INVALID; }
    ctx->peer = true;
  }
  if (opt && (opt->flags & 4) && !dist) { set_err(ctx, "options.flags bit2 needs a distributed ctx"); return PLSS_E_INVALID; }
  if (opt && (opt->flags & 4) && ctx->nranks > 64) { set_err(ctx, "reduce-scatter step: at most 64 ranks"); return PLSS_E_INVALID; }
  if (dist && opt && (opt->flags & 4)) {
    ctx->rsag = true;
    ctx->cnt = (A->n + ctx->nranks - 1) / ctx->nranks;
    ctx->cnt = (ctx->cnt + 31) / 32 * 32;
    ctx->c0 = (int64_t)ctx->rank * ctx->cnt;
    ctx->nsh = std::max<int64_t>(0, std::min<int64_t>(A->n, ctx->c0 + ctx->cnt) - ctx->c0);
  }
  {
    const void* arrs[6] = {A->row_ptr, A->col_idx, A->val, A->col_ptr, A->row_idx, A->val_t};
    for (const void* q : arrs)
      if (q && (reinterpret_cast<uintptr_t>(q) & 15) != 0) {
        set_err(ctx, "matrix arrays must be 16-byte aligned (TMA bulk copies)");
        return PLSS_E_INVALID;
      }
  }
  CK(cudaGetDevice(&ctx->dev));
  ctx->user_stream = (cudaStream_t)stream;
  if (ctx->user_stream == nullptr) {
    // the legacy default stream cannot be captured into a graph: work on our own stream and
    // order it against the caller's stream with events (sync_in / sync_out)
    CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    ctx->own_stream = true;
  } else {
    ctx->stream = ctx->user_stream;
  }
  CK(cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_out, cudaEventDisableTiming));
  CK(cudaStreamSynchronize(ctx->user_stream));
  cudaStream_t st = ctx->stream;
  const Layout& L = ctx->L;
  ctx->S = L.S;
  ctx->ws = (char*)workspace;
  char* w = ctx->ws;
  ctx->r = (double*)(w + L.r); ctx->y = (double*)(w + L.y); ctx->p = (double*)(w + L.p);
  ctx->x = (double*)(w + L.x); ctx->rec = (double*)(w + L.rec); ctx->ctl = (Ctl*)(w + L.ctl);
  ctx->counters = (unsigned*)(w + L.counters);
  ctx->part1 = (double*)(w + L.part1); ctx->part2 = (double*)(w + L.part2);
  ctx->part3 = (double*)(w + L.part3); ctx->partn = (double*)(w + L.partn);
  ctx->scalars = (double*)(w + L.scalars);
  ctx->wi = (double*)(w + L.wi);
  int* d_err = (int*)(w + L.err);
  if (ctx->peer) {
    ctx->sym_yb = align_up(8 * (size_t)(A->n + 2));
    const size_t bytes = 2 * ctx->sym_yb + 4 * (size_t)PF_WORDS;
    CK(cudaMalloc((void**)&ctx->sym, bytes));
    CK(cudaMemsetAsync(ctx->sym, 0, bytes, ctx->stream ? ctx->stream : nullptr));
    ctx->yred = (double*)ctx->sym;
    ctx->y = (double*)(ctx->sym + ctx->sym_yb);
  }
  CK(cudaMemsetAsync(ctx->counters, 0, 64 * sizeof(unsigned), st));
  CK(cudaMemsetAsync(ctx->part1, 0, 16 * (size_t)MAXG * L.S, st));
  CK(cudaMemsetAsync(ctx->part2, 0, 16 * (size_t)MAXG, st));
  CK(cudaMemsetAsync(ctx->part3, 0, 16 * (size_t)MAXG, st));
  CK(cudaMemsetAsync(ctx->ctl, 0, sizeof(Ctl), st));
  CK(cudaMemsetAsync(d_err, 0, 64, st));

  const int64_t m = ctx->m, n = ctx->n, nnz = ctx->nnz;
  // ---- validation --------------------------------------------------------------------------
  if (A->validate) {
    const int bs = 256;
    k_validate<<<(unsigned)((std::max<int64_t>(m, 1) + bs - 1) / bs), bs, 0, st>>>(A->row_ptr, A->col_idx, A->val, m, n, nnz, d_err);
    k_validate<<<(unsigned)((std::max<int64_t>(n, 1) + bs - 1) / bs), bs, 0, st>>>(A->col_ptr, A->row_idx, A->val_t, n, m, nnz, d_err + 1);
    CK(cudaGetLastError());
    int h_err[2] = {0, 0};
    CK(cudaMemcpyAsync(h_err, d_err, sizeof(h_err), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h_err[0] || h_err[1]) {
      char buf[128];
      snprintf(buf, sizeof buf, "matrix format violation (csr flags %d, csc flags %d)", h_err[0], h_err[1]);
      set_err(ctx, buf);
      return PLSS_E_FORMAT;
    }
    if (n > 0)
      k_validate_pair<<<(unsigned)((n + bs - 1) / bs), bs, 0, st>>>(A->row_ptr, A->col_idx, A->val, A->col_ptr, A->row_idx, A->val_t, n, d_err + 2);
    CK(cudaGetLastError());
    int h2 = 0;
    CK(cudaMemcpyAsync(&h2, d_err + 2, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h2) { set_err(ctx, "CSC copy is not the transpose of the CSR matrix"); return PLSS_E_FORMAT; }
  }

  // ---- slab bounds ---------------------------------------------------------------------------
  const int S = ctx->S;
  ctx->R.resize(S + 1);
  ctx->E.resize(S + 1);
  for (int s = 0; s <= S; ++s) ctx->R[s] = (m * s) / S;
  {
    std::vector<int32_t> tmp(S + 1);
    for (int s = 0; s <= S; ++s)
      CK(cudaMemcpyAsync(&tmp[s], A->row_ptr + ctx->R[s], sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int s = 0; s <= S; ++s) ctx->E[s] = tmp[s];
    if (ctx->E[0] != 0 || ctx->E[S] != nnz) { set_err(ctx, "row_ptr[0] != 0 or row_ptr[m] != nnz"); return PLSS_E_FORMAT; }
  }

  // ---- occupancy-derived persistent grids -----------------------------------------------------
  int sms = 0, occ_vec = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->dev));
  int occ[4] = {0, 0, 0, 0};
  if (set_smem_attrs(ctx, occ) != PLSS_OK) return PLSS_E_CUDA;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_vec, k_pxupdate, NT, 0));
  occ_vec = std::max(1, occ_vec);
  int occ_sell = 1;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_sell, k_sell<ROLE_K2DOTS>, NT, 0));
  occ_sell = std::max(1, occ_sell);
  SellPool pool1{}, pool2{};
  if (L.sell) {
    pool1 = SellPool{(int32_t*)(w + L.s1idx), (int32_t*)(w + L.s1perm), (int32_t*)(w + L.s1sptr),
                     (double*)(w + L.s1val), L.s1cap, L.s1slots, L.s1sp, 0, 0, 0,
                     (int2*)(w + L.s1win), L.s1sp / 4 + 2 * S + 2, 0, (int32_t*)(w + L.cblk), 0,
                     (int32_t*)(w + L.s1aux), L.s1auxn, 0};
    pool2 = SellPool{(int32_t*)(w + L.s2idx), (int32_t*)(w + L.s2perm), (int32_t*)(w + L.s2sptr),
                     (double*)(w + L.s2val), L.s2cap, L.s2slots, L.s2sp, 0, 0, 0,
                     (int2*)(w + L.s2win), L.s2sp / 4 + 2 * S + 2, 0,
                     (int32_t*)(w + L.cblk) + (size_t)(MAXG + 1) * S, 0,
                     (int32_t*)(w + L.s2aux), L.s2auxn, 0};
    // windowed kernels: up to ~200 KB of dynamic shared memory for the ring
    CK(cudaFuncSetAttribute(k_sellw<ROLE_PLAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_sellw<ROLE_K1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_sellw<ROLE_K2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_sellw<ROLE_K2DOTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_win_choose, cudaFuncAttributeMaxDynamicSharedMemorySize, 16385 * 4));
    CK(cudaFuncSetAttribute(k_sell<ROLE_K2, 1024, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            YSTAGE_SMEM));
    CK(cudaFuncSetAttribute(k_sell<ROLE_K2DOTS, 1024, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            YSTAGE_SMEM));
    CK(cudaFuncSetAttribute(k_sell<ROLE_K2, 1024, false, true, SIGMA_WIDE>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, YSTAGE_SMEM_WIDE));
    CK(cudaFuncSetAttribute(k_sell<ROLE_K2DOTS, 1024, false, true, SIGMA_WIDE>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, YSTAGE_SMEM_WIDE));
  }
  // Shared-memory windows (fmt 2) are opt-in: correct and bit-exact, but on every config measured
  // slower than L1-cached gathers ("Windows"). opt.flags bit1 disables them
  // even when requested through PLSS_WIN1 / PLSS_WIN2 (window lengths in doubles).
  const int win1 = L.window ? env_int("PLSS_WIN1", 0) : 0;       // window of p (K1)
  const int win2 = L.window ? env_int("PLSS_WIN2", 0) : 0;       // window of r_s (K2)
  // fmt 3 (one 1024-thread CTA per SM over a contiguous entry-balanced slice range, warps taking
  // slices in order): default for K1 and K2 (C5: K1 2.6-2.7 vs 2.9-3.0 ms, K2 4.06 vs 4.66 ms with
  // fmt 1). PLSS_SELLC: 0 off, 1 K1 only, 2 K1 + K2.
  const int contig = env_int("PLSS_SELLC", 2);
  const int nsb1 = env_int("PLSS_NSB1", 16), nsb2 = env_int("PLSS_NSB2", 8);   // slices per window block
  auto sell_grid = [&](const SpmvSeg& a) {
    return grid_for(((int64_t)a.nslices + NT / 32 - 1) / (NT / 32), occ_sell, sms);
  };

  // ---- L2 cache policies (uniform kernel parameters, see SpmvSeg::pol_first) -------------------
  uint64_t pols[2] = {0, 0};
  {
    uint64_t* d_pol = (uint64_t*)(w + L.err + 32);
    k_policies<<<1, 1, 0, st>>>(d_pol);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(pols, d_pol, sizeof pols, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }

  // ---- K1 segments (CSR row slabs) ----------------------------------------------------------
  int2* desc1 = (int2*)(w + L.tile1);
  int2* desc2 = (int2*)(w + L.tile2);
  const int64_t tiles1_cap = (int64_t)((L.tile2 - L.tile1) / 8);
  const int64_t tiles2_cap = (int64_t)((L.scratch - L.tile2) / 8);
  int64_t t1off = 0, t2off = 0;
  ctx->seg1.resize(S);
  ctx->seg2.resize(S);
  ctx->g1.resize(S);
  ctx->g2.resize(S);
  for (int s = 0; s < S; ++s) {
    SpmvSeg& a = ctx->seg1[s];
    memset(&a, 0, sizeof a);
    a.pol_first = pols[0];
    a.pol_last = pols[1];
    const int64_t rows = ctx->R[s + 1] - ctx->R[s];
    a.ptr = A->row_ptr + ctx->R[s];
    a.idx = A->col_idx;
    a.val = A->val;
    a.desc = desc1 + t1off;
    a.e0 = ctx->E[s];
    a.nrows = (int32_t)rows;
    a.row0 = (int32_t)ctx->R[s];
    int64_t nt = 0;
    if (build_tiles(ctx, a.ptr, rows, a.e0, (int2*)a.desc, tiles1_cap - t1off, &nt) != PLSS_OK) return PLSS_E_CUDA;
    a.ntiles = (int32_t)nt;
    a.g = ctx->p;
    a.out = ctx->r + ctx->R[s];
    a.partial = ctx->part1 + 2 * (size_t)MAXG * s;
    a.part_base = ctx->part1;
    a.nparts = MAXG * S;
    a.finalize = (s == S - 1);
    a.dist = dist ? 1 : 0;
    a.counter = ctx->counters + 0;
    a.ctl = ctx->ctl;
    a.rec = ctx->rec;
    a.rho_out = ctx->rsag ? ctx->scalars + 4 : ctx->cols ? ctx->scalars + 8 : ctx->y + n;
    t1off += nt + 1;
    ctx->g1[s] = grid_for(nt, occ[ROLE_K1], sms);
    if (L.sell) {
      if (try_sell(ctx, a, ctx->E[s + 1] - ctx->E[s], pool1, sms, occ_sell) != PLSS_OK) return PLSS_E_CUDA;
      if (a.fmt == 1) ctx->g1[s] = sell_grid(a);
      if (try_window(ctx, a, ctx->p, n, ctx->E[s + 1] - ctx->E[s], win1, nsb1, pool1, sms, &ctx->g1[s]) != PLSS_OK)
        return PLSS_E_CUDA;
      if ((contig >= 1 || a.gsort) && make_contig(ctx, a, pool1, sms, &ctx->g1[s]) != PLSS_OK) return PLSS_E_CUDA;
    }
  }

  // ---- K2 segments (CSC, slab-major copy when S > 1) ----------------------------------------
  int32_t *sptr = nullptr, *sidx = nullptr;
  double* sval = nullptr;
  if (S > 1) {
    if (L.sell) {
      // setup-time slab-major CSC (9.5 GB for C5): freed below unless a K2 segment keeps reading it
      const size_t b_sptr = align_up(4 * (size_t)S * (n + 1)), b_sidx = align_up(4 * (size_t)std::max<int64_t>(nnz, 1));
      const size_t bytes = b_sptr + b_sidx + 8 * (size_t)std::max<int64_t>(nnz, 1);
      CK(cudaMalloc((void**)&ctx->slabmajor, bytes));
      sptr = (int32_t*)ctx->slabmajor;
      sidx = (int32_t*)(ctx->slabmajor + b_sptr);
      sval = (double*)(ctx->slabmajor + b_sptr + b_sidx);
    } else {
      sptr = (int32_t*)(w + L.sptr);
      sidx = (int32_t*)(w + L.sidx);
      sval = (double*)(w + L.sval);
    }
    int32_t* blk = (int32_t*)(w + L.scan_blk);
    const long long len = n + 1;
    for (int s = 0; s < S; ++s) {
      int32_t* sp = sptr + (size_t)s * (n + 1);
      k_slab_count<<<(unsigned)((len + 255) / 256), 256, 0, st>>>(A->col_ptr, A->row_idx, n, ctx->R[s], ctx->R[s + 1], sp);
      if (scan_excl(ctx, sp, len, blk) != PLSS_OK) return PLSS_E_CUDA;
      k_slab_copy<<<(unsigned)((len + 255) / 256), 256, 0, st>>>(A->col_ptr, A->row_idx, A->val_t, n, ctx->R[s], ctx->R[s + 1], ctx->E[s], sp, sidx, sval);
    }
    CK(cudaGetLastError());
  }
  for (int s = 0; s < S; ++s) {
    SpmvSeg& a = ctx->seg2[s];
    memset(&a, 0, sizeof a);
    a.pol_first = pols[0];
    a.pol_last = pols[1];
    if (S > 1) {
      a.ptr = sptr + (size_t)s * (n + 1);
      a.idx = sidx;
      a.val = sval;
      a.e0 = ctx->E[s];
      a.g = ctx->r + ctx->R[s];
    } else {
      a.ptr = A->col_ptr;
      a.idx = A->row_idx;
      a.val = A->val_t;
      a.e0 = 0;
      a.g = ctx->r;
    }
    a.desc = desc2 + t2off;
    a.nrows = (int32_t)n;
    a.row0 = (int32_t)ctx->R[s];
    int64_t nt = 0;
    if (build_tiles(ctx, a.ptr, n, a.e0, (int2*)a.desc, tiles2_cap - t2off, &nt) != PLSS_OK) return PLSS_E_CUDA;
    a.ntiles = (int32_t)nt;
    a.out = ctx->y;
    a.pv = ctx->p;
    a.wi = ctx->wi;
    a.partial = ctx->part2;
    a.part_base = ctx->part2;
    a.nparts = MAXG;
    a.accumulate = (s > 0);
    a.finalize = (!dist && s == S - 1);
    a.psi3 = (a.finalize && env_int("PLSS_PSI3", 1)) ? 1 : 0;   // psi summed by K3 (k2_final)
    a.counter = ctx->counters + 1;
    a.ctl = ctx->ctl;
    a.rec = ctx->rec;
    t2off += nt + 1;
    ctx->g2[s] = grid_for(nt, occ[a.finalize ? ROLE_K2DOTS : ROLE_K2], sms);
    if (L.sell) {
      if (try_scalar(ctx, a, ctx->E[s + 1] - ctx->E[s], sms, &ctx->g2[s]) != PLSS_OK) return PLSS_E_CUDA;
      if (a.fmt == 0 &&
          try_sell(ctx, a, ctx->E[s + 1] - ctx->E[s], pool2, sms, occ_sell, win2 == 0 && env_int("PLSS_SIGWIDE", 1))
          != PLSS_OK)
        return PLSS_E_CUDA;
      if (a.fmt == 1) ctx->g2[s] = sell_grid(a);
      if (try_window(ctx, a, a.g, ctx->R[s + 1] - ctx->R[s], ctx->E[s + 1] - ctx->E[s], win2, nsb2, pool2, sms,
                     &ctx->g2[s]) != PLSS_OK)
        return PLSS_E_CUDA;
      if ((contig >= 2 || a.gsort) && make_contig(ctx, a, pool2, sms, &ctx->g2[s]) != PLSS_OK) return PLSS_E_CUDA;
    }
  }
  CK(cudaGetLastError());
  // Diagnostics: per-CTA timing of the fmt 3 launches (plss_debug_cta_times)
  if (env_int("PLSS_DBG_CTA", 0)) {
    for (int s = 0; s < S; ++s)
      for (SpmvSeg* a : {&ctx->seg1[s], &ctx->seg2[s]}) {
        CK(cudaMalloc((void**)&a->ctat, 4 * 8 * (size_t)MAXG));
        CK(cudaMemsetAsync(a->ctat, 0, 4 * 8 * (size_t)MAXG, st));
        ctx->dbg_bufs.push_back(a->ctat);
      }
  }
  // Static stepping (SpmvSeg::stat) for fmt 3 segments without a perm or long rows (C5's K1:
  // 2.78 -> 2.61 ms per step), with 6 entries in flight per lane when the slices are 6k steps long
  // (C5's K1 rows of 12: 2.61 -> 2.52 ms; K2's variable columns keep 8). PLSS_STAT=0 turns it off.
  {
    const int stat = env_int("PLSS_STAT", 1);
    for (int s = 0; s < S; ++s) {
      for (SpmvSeg* a : {&ctx->seg1[s], &ctx->seg2[s]}) {
        a->stat = (stat && a->fmt == 3 && !a->perm && !a->gsort) ? 1 : 0;
        if (a->stat && a->nslices > 0) {
          int32_t ends[2] = {0, 0};                  // sptr[0], sptr[nslices]: all slices of equal length?
          CK(cudaMemcpyAsync(&ends[0], a->sptr, 4, cudaMemcpyDeviceToHost, st));
          CK(cudaMemcpyAsync(&ends[1], a->sptr + a->nslices, 4, cudaMemcpyDeviceToHost, st));
          CK(cudaStreamSynchronize(st));
          const int64_t tot = (int64_t)ends[1] - ends[0];
          if (tot % a->nslices == 0 && (tot / a->nslices) % 6 == 0 && stat != 3) a->stat = 2;
        }
      }
    }
  }
  if (dist && L.sell && !ctx->rsag && !ctx->cols) {
    const plss_status st2 = make_chunks(ctx, ctx->seg2[S - 1], pool2, sms, env_int("PLSS_DIST_CHUNKS", 4));
    if (st2 != PLSS_OK) return st2;
  }
  // k_longrows' fork / join (launch_spmv): one non-blocking stream and two events per ctx
  if (env_int("PLSS_FORK", 1)) {
    bool any = false;
    for (auto* v : {&ctx->seg1, &ctx->seg2}) for (auto& a : *v) any |= a.fmt == 3 && a.nlong > 0;
    if (any) {
      CK(cudaStreamCreateWithFlags(&ctx->fork_stream, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming));
      for (auto* v : {&ctx->seg1, &ctx->seg2})
        for (auto& a : *v)
          if (a.fmt == 3 && a.nlong > 0) { a.fork_stream = ctx->fork_stream; a.fork_ev = ctx->fork_ev; a.join_ev = ctx->join_ev; }
    }
  }
  // release the setup-time slab-major CSC when no K2 segment reads it after setup: SELL formats read
  // their own copies; CSR tiles (fmt 0), a thread per column (fmt 5) and the long rows of a globally
  // sorted segment (k_longrows) read the slab-major arrays
  if (ctx->slabmajor) {
    bool keep = false;
    for (auto& a : ctx->seg2) keep |= a.fmt == 0 || a.fmt == 5 || (a.gsort && a.nlong > 0);
    if (!keep) {
      CK(cudaStreamSynchronize(st));
      CK(cudaFree(ctx->slabmajor));
      ctx->slabmajor = nullptr;
      for (auto& a : ctx->seg2) { a.ptr = nullptr; a.desc = nullptr; }   // not read by the SELL formats
    }
  }
  // One slab on one device: the finalizing sums need only the partial slots the launch writes
  // (grid, + 1 for a globally sorted segment's long rows); the other slots hold zeros, so the
  // totals are bitwise the same and the electing CTA (or k_longchunks' warp) reads ~150 pairs
  // instead of MAXG
  if (!dist && S == 1) {
    ctx->seg1[0].nparts = std::min(MAXG, ctx->g1[0] + 1);
    ctx->seg2[0].nparts = std::min(MAXG, ctx->g2[0] + 1);
  }
  ctx->xdefer = !ctx->cols && !ctx->rsag && env_int("PLSS_XDEFER", 1);
  ctx->psi_dots = (dist && !ctx->cols && !ctx->rsag && env_int("PLSS_PSI3", 1)) ? 1 : 0;
  ctx->g3 = grid_for((n / 2 + NT - 1) / NT + 1, occ_vec, sms);
  ctx->gdots = grid_for((n + NT - 1) / NT + 1, occ_vec, sms);
  ctx->gnorm = grid_for((m + NT - 1) / NT + 1, occ_vec, sms);

  CK(cudaHostAlloc((void**)&ctx->h_done, 2 * sizeof(int32_t), cudaHostAllocDefault));
  CK(cudaHostAlloc((void**)&ctx->h_ctl, sizeof(Ctl), cudaHostAllocDefault));
  CK(cudaEventCreateWithFlags(&ctx->ev[0], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev[1], cudaEventDisableTiming));
  ctx->chunk = (opt && opt->graph_chunk > 0) ? opt->graph_chunk : 16;
  CK(cudaStreamSynchronize(st));
  return PLSS_OK;
}

// peer-memory step: map every rank's region (CUDA IPC handles, all-gathered over the ctx's own
// communicator) and size the reduce grid
static plss_status peer_connect(plss_ctx* ctx) {
  const int G = ctx->nranks;
  cudaStream_t st = ctx->stream;
  std::vector<cudaIpcMemHandle_t> hs(G);
  if (G > 1) {
    const size_t hb = sizeof(cudaIpcMemHandle_t);
    CK(cudaIpcGetMemHandle(&hs[ctx->rank], ctx->sym));
    char* d = nullptr;
    CK(cudaMallocAsync((void**)&d, hb * G, st));
    CK(cudaMemcpyAsync(d + hb * ctx->rank, &hs[ctx->rank], hb, cudaMemcpyHostToDevice, st));
    NK(ncclAllGather(d + hb * ctx->rank, d, hb, ncclUint8, ctx->comm, st));
    CK(cudaMemcpyAsync(hs.data(), d, hb * G, cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(d, st));
    CK(cudaStreamSynchronize(st));
  }
  for (int h = 0; h < G; ++h) {
    char* base = ctx->sym;
    if (h != ctx->rank) {
      void* q = nullptr;
      CK(cudaIpcOpenMemHandle(&q, hs[h], cudaIpcMemLazyEnablePeerAccess));
      ctx->ipc_open.push_back(q);
      base = (char*)q;
    }
    ctx->ptab.red[h] = (double*)base;
    ctx->ptab.part[h] = (const double*)(base + ctx->sym_yb);
    ctx->ptab.flg[h] = (unsigned*)(base + 2 * ctx->sym_yb);
  }
  int sms = 1;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->dev));
  const int64_t per = (ctx->n + 1) / peer_nch(ctx) / G + 2;              // shard of a chunk
  int occ = 1;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_peer_reduce, PEER_NT, 0));
  const int cap = std::max(1, occ) * sms;                              // co-resident (see k_peer_reduce)
  const int gx = env_int("PLSS_PEER_GX", 0);
  ctx->peer_gx = gx > 0 ? std::min(gx, cap)
                        : (int)std::max<int64_t>(1, std::min<int64_t>((per / 4 + PEER_NT - 1) / PEER_NT, cap));
  return PLSS_OK;
}

static plss_status finish_create(plss_ctx* ctx) {
  // graphs are captured after setup so their nodes carry the final kernel parameters
  // (the device state they read is reset by plss_start); capture does not execute kernels
  plss_status st = build_graph(ctx, ctx->chunk, &ctx->graph_chunk);
  if (st != PLSS_OK) return st;
  st = build_graph(ctx, 1, &ctx->graph_one);
  if (st != PLSS_OK) return st;
  CK(cudaStreamSynchronize(ctx->stream));
  return PLSS_OK;
}

extern "C" {

size_t plss_workspace_bytes(const plss_matrix* A, const plss_options* opt) {
  Layout L;
  if (!compute_layout(A, opt, false, &L)) return 0;
  return L.total;
}

plss_status plss_create(const plss_matrix* A, const plss_options* opt, void* workspace, size_t ws_bytes,
                        void* cuda_stream, plss_ctx** out) {
  NvtxRange nvtx_("plss_create");
  if (!A || !out) { g_last_error = "NULL argument"; return PLSS_E_INVALID; }
  *out = nullptr;
  plss_ctx* ctx = new (std::nothrow) plss_ctx();
  if (!ctx) return PLSS_E_NOMEM;
  plss_status st = setup(ctx, A, opt, workspace, ws_bytes, cuda_stream, false);
  if (st == PLSS_OK) st = finish_create(ctx);
  if (st != PLSS_OK) { g_last_error = ctx->err; plss_destroy(ctx); return st; }
  *out = ctx;
  return PLSS_OK;
}

plss_status plss_get_unique_id(uint8_t id[128]) {
  if (!id) return PLSS_E_INVALID;
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) { g_last_error = ncclGetErrorString(r); return PLSS_E_NCCL; }
  static_assert(sizeof(u) == 128, "ncclUniqueId size");
  memcpy(id, &u, 128);
  return PLSS_OK;
}

plss_status plss_create_dist(const plss_matrix* A_local, int64_t row_offset, int64_t m_global,
                             const uint8_t id[128], int32_t rank, int32_t nranks, const plss_options* opt,
                             void* workspace, size_t ws_bytes, void* cuda_stream, plss_ctx** out) {
  NvtxRange nvtx_("plss_create_dist");
  if (!A_local || !out || !id || nranks < 1 || rank < 0 || rank >= nranks) { g_last_error = "invalid argument"; return PLSS_E_INVALID; }
  if (row_offset < 0 || row_offset + A_local->m > m_global) { g_last_error = "row block outside the global matrix"; return PLSS_E_DIM; }
  *out = nullptr;
  plss_ctx* ctx = new (std::nothrow) plss_ctx();
  if (!ctx) return PLSS_E_NOMEM;
  ctx->rank = rank;
  ctx->nranks = nranks;
  ctx->dist = true;
  ctx->row_offset = row_offset;
  ctx->m_global = m_global;
  ctx->fault_nccl = env_int("PLSS_FAULT_NCCL", 0);
  ctx->wait_timeout_s = env_int("PLSS_WAIT_TIMEOUT_S", 600);
  plss_status st = setup(ctx, A_local, opt, workspace, ws_bytes, cuda_stream, true);
  if (st == PLSS_OK) {
    ncclUniqueId u;
    memcpy(&u, id, 128);
    ncclResult_t r = ncclCommInitRank(&ctx->comm, nranks, u, rank);
    if (r != ncclSuccess) { set_err(ctx, std::string("ncclCommInitRank: ") + ncclGetErrorString(r)); st = PLSS_E_NCCL; }
  }
  if (st == PLSS_OK && ctx->peer) st = peer_connect(ctx);
  if (st == PLSS_OK) st = finish_create(ctx);
  if (st != PLSS_OK) { g_last_error = ctx->err; plss_destroy(ctx); return st; }
  *out = ctx;
  return PLSS_OK;
}

plss_status plss_create_dist_cols(const plss_matrix* A_local, int64_t col_offset, int64_t n_global,
                                  const uint8_t id[128], int32_t rank, int32_t nranks, const plss_options* opt,
                                  void* workspace, size_t ws_bytes, void* cuda_stream, plss_ctx** out) {
  NvtxRange nvtx_("plss_create_dist_cols");
  if (!A_local || !out || !id || nranks < 1 || rank < 0 || rank >= nranks) { g_last_error = "invalid argument"; return PLSS_E_INVALID; }
  if (col_offset < 0 || col_offset + A_local->n > n_global) { g_last_error = "column block outside the global matrix"; return PLSS_E_DIM; }
  if (opt && (opt->flags & 12)) { g_last_error = "options.flags bit2 / bit3 are row-block steps"; return PLSS_E_INVALID; }
  *out = nullptr;
  plss_ctx* ctx = new (std::nothrow) plss_ctx();
  if (!ctx) return PLSS_E_NOMEM;
  ctx->rank = rank;
  ctx->nranks = nranks;
  ctx->dist = true;
  ctx->cols = true;
  ctx->col_offset = col_offset;
  ctx->n_global = n_global;
  ctx->fault_nccl = env_int("PLSS_FAULT_NCCL", 0);
  ctx->wait_timeout_s = env_int("PLSS_WAIT_TIMEOUT_S", 600);
  plss_status st = setup(ctx, A_local, opt, workspace, ws_bytes, cuda_stream, true);
  if (st == PLSS_OK) {
    ncclUniqueId u;
    memcpy(&u, id, 128);
    ncclResult_t r = ncclCommInitRank(&ctx->comm, nranks, u, rank);
    if (r != ncclSuccess) { set_err(ctx, std::string("ncclCommInitRank: ") + ncclGetErrorString(r)); st = PLSS_E_NCCL; }
  }
  if (st == PLSS_OK) st = finish_create(ctx);
  if (st != PLSS_OK) { g_last_error = ctx->err; plss_destroy(ctx); return st; }
  *out = ctx;
  return PLSS_OK;
}

// Wait for an event (or, ev = NULL, the stream). On a distributed ctx the wait polls the
// communicator's asynchronous error state (failure detection): on an error -- or after
// PLSS_WAIT_TIMEOUT_S seconds (default 600) without completion, e.g. a rank that died before its
// collective -- the communicator is aborted (ncclCommAbort makes the pending collectives return),
// the call fails with PLSS_E_NCCL and the ctx stays unusable until plss_destroy.
static plss_status dist_wait(plss_ctx* ctx, cudaStream_t st, cudaEvent_t ev) {
  NvtxRange nvtx_("plss: wait (stream / NCCL async-error poll)");
  if (!ctx->dist || !ctx->comm) {
    if (ev) CK(cudaEventSynchronize(ev)); else CK(cudaStreamSynchronize(st));
    return PLSS_OK;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (int spin = 0;; ++spin) {
    const cudaError_t q = ev ? cudaEventQuery(ev) : cudaStreamQuery(st);
    if (q != cudaSuccess && q != cudaErrorNotReady) CK(q);
    ncclResult_t a = ncclSuccess;
    const ncclResult_t r = ncclCommGetAsyncError(ctx->comm, &a);
    if (ctx->fault_nccl) a = ncclSystemError;
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const bool timeout = ctx->wait_timeout_s > 0 && el > ctx->wait_timeout_s;
    if (r != ncclSuccess || (a != ncclSuccess && a != ncclInProgress) || timeout) {
      ncclCommAbort(ctx->comm);
      ctx->comm = nullptr;
      ctx->aborted = true;
      cudaStreamSynchronize(st);                     // the aborted collectives return
      cudaGetLastError();
      set_err(ctx, timeout ? std::string("collective did not complete within PLSS_WAIT_TIMEOUT_S; communicator aborted")
                           : std::string("NCCL asynchronous error: ") + ncclGetErrorString(r != ncclSuccess ? r : a) +
                                 "; communicator aborted");
      return PLSS_E_NCCL;
    }
    if (q == cudaSuccess) return PLSS_OK;
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

static plss_status check_live(plss_ctx* ctx) {
  if (ctx->aborted) { set_err(ctx, "the communicator was aborted after an NCCL failure; destroy the ctx"); return PLSS_E_NCCL; }
  return PLSS_OK;
}

plss_status plss_start(plss_ctx* ctx, const double* b, const double* x0, double tol, int32_t tol_mode,
                       int32_t maxit, int32_t flags) {
  NvtxRange nvtx_("plss_start");
  if (!ctx) return PLSS_E_INVALID;
  if (check_live(ctx) != PLSS_OK) return PLSS_E_NCCL;
  if (!(tol >= 0.0) || maxit < 1 || maxit > ctx->L.maxit_cap || (tol_mode != 0 && tol_mode != 1) ||
      (flags & ~1) != 0) {
    set_err(ctx, "invalid tol / tol_mode / maxit / flags");
    return PLSS_E_INVALID;
  }
  if (!b && ctx->m > 0) { set_err(ctx, "b is NULL"); return PLSS_E_INVALID; }
  cudaStream_t st = ctx->stream;
  if (sync_in(ctx) != PLSS_OK) return PLSS_E_CUDA;
  const int64_t m = ctx->m, n = ctx->n;
  Ctl& c = *ctx->h_ctl;
  memset(&c, 0, sizeof c);
  c.nbd = 1.0;
  c.tol = tol;
  c.freeze_h = 64.0 * 2.220446049250313e-16;
  c.maxit = maxit;
  c.freeze = flags & 1;
  c.tol_mode = tol_mode;
  c.weighted = ctx->weighted ? 1 : 0;
  c.outcome = OUT_RUNNING;
  CK(cudaMemcpyAsync(ctx->ctl, &c, sizeof(Ctl), cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(ctx->rec, 0, 8 * (size_t)(maxit + 1) * REC, st));
  if (m > 0) CK(cudaMemcpyAsync(ctx->r, b, 8 * (size_t)m, is_device_ptr(b) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  if (n > 0) {
    if (x0) {
      const cudaMemcpyKind kind = is_device_ptr(x0) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
      CK(cudaMemcpyAsync(ctx->p, x0, 8 * (size_t)n, kind, st));   // K1 of step 0 gathers x0: r = b - A x0
      CK(cudaMemcpyAsync(ctx->x, x0, 8 * (size_t)n, kind, st));
    } else {
      CK(cudaMemsetAsync(ctx->p, 0, 8 * (size_t)n, st));
      CK(cudaMemsetAsync(ctx->x, 0, 8 * (size_t)n, st));
    }
  }
  if (ctx->rsag) {                                  // padding beyond n of the reduce-scattered y and of p
    const size_t pad = (size_t)(ctx->cnt * ctx->nranks - n);
    CK(cudaMemsetAsync(ctx->y + n, 0, 8 * (pad + 1), st));
    CK(cudaMemsetAsync(ctx->p + n, 0, 8 * pad, st));
    CK(cudaMemsetAsync(ctx->scalars + 4, 0, 32, st));
  }
  if (ctx->cols) {
    // b is replicated: ||b|| locally (the same bytes, the same sum on every rank); then the
    // all-reduced u of the first K1 must sum to b - A x0: ranks > 0 start from u = 0
    k_norm_b<<<ctx->gnorm, NT, 0, st>>>(ctx->r, m, ctx->ctl, ctx->partn, ctx->counters + 3, 1, nullptr);
    if (ctx->rank > 0 && m > 0) CK(cudaMemsetAsync(ctx->r, 0, 8 * (size_t)m, st));
    CK(cudaMemsetAsync(ctx->r + m, 0, 8, st));
  } else if (ctx->dist) {
    k_norm_b<<<ctx->gnorm, NT, 0, st>>>(ctx->r, m, ctx->ctl, ctx->partn, ctx->counters + 3, 0, ctx->scalars);
    CK(cudaGetLastError());
    NK(ncclAllReduce(ctx->scalars, ctx->scalars, 1, ncclFloat64, ncclSum, ctx->comm, st));
    k_set_nbd<<<1, 1, 0, st>>>(ctx->ctl, ctx->scalars);
  } else {
    k_norm_b<<<ctx->gnorm, NT, 0, st>>>(ctx->r, m, ctx->ctl, ctx->partn, ctx->counters + 3, 1, nullptr);
  }
  CK(cudaGetLastError());
  ctx->started = true;
  ctx->rp_started = false;
  ctx->kz_started = false;
  ctx->eg_started = false;
  ctx->maxit = maxit;
  ctx->flags = flags;
  return PLSS_OK;
}

plss_status plss_step(plss_ctx* ctx, int32_t k) {
  NvtxRange nvtx_("plss_step");
  if (!ctx) return PLSS_E_INVALID;
  if (check_live(ctx) != PLSS_OK) return PLSS_E_NCCL;
  if (!ctx->started) { set_err(ctx, "plss_step before plss_start"); return PLSS_E_STATE; }
  if (k < 0) return PLSS_E_INVALID;
  for (int i = 0; i + ctx->chunk <= k; i += ctx->chunk) CK(cudaGraphLaunch(ctx->graph_chunk, ctx->stream));
  for (int i = 0; i < k % ctx->chunk; ++i) CK(cudaGraphLaunch(ctx->graph_one, ctx->stream));
  return PLSS_OK;
}

plss_status plss_finish(plss_ctx* ctx, double* x, int32_t* iters, double* hist, double* diag,
                        plss_outcome* outcome) {
  NvtxRange nvtx_("plss_finish");
  if (!ctx) return PLSS_E_INVALID;
  if (check_live(ctx) != PLSS_OK) return PLSS_E_NCCL;
  if (!ctx->started) { set_err(ctx, "plss_finish before plss_start"); return PLSS_E_STATE; }
  cudaStream_t st = ctx->stream;
  if (ctx->rsag)                                    // x lives as column shards: gather (collective)
    NK(ncclAllGather(ctx->x + ctx->c0, ctx->x, (size_t)ctx->cnt, ncclFloat64, ctx->comm, st));
  if (ctx->xdefer && ctx->n > 0) {                  // x lags one update (K3_XDEFER): x <- x + p
    k_xflush<<<ctx->g3, NT, 0, st>>>(ctx->x, ctx->p, ctx->n, ctx->ctl);
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(&ctx->ctl->xlag, 0, sizeof(int32_t), st));
  }
  if (x && ctx->n > 0)
    CK(cudaMemcpyAsync(x, ctx->x, 8 * (size_t)ctx->n, is_device_ptr(x) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(ctx->h_ctl, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
  std::vector<double> rec;
  if (hist || diag) {
    rec.resize((size_t)(ctx->maxit + 1) * REC);
    CK(cudaMemcpyAsync(rec.data(), ctx->rec, 8 * rec.size(), cudaMemcpyDeviceToHost, st));
  }
  unsigned peer_err = 0;
  if (ctx->peer)
    CK(cudaMemcpyAsync(&peer_err, ctx->ptab.flg[ctx->rank] + PF_ERR, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  {
    const plss_status w = dist_wait(ctx, st, nullptr);
    if (w != PLSS_OK) return w;
  }
  if (sync_out(ctx) != PLSS_OK) return PLSS_E_CUDA;
  if (peer_err) { set_err(ctx, "peer-memory step: a rank did not arrive within 20 s"); return PLSS_E_CUDA; }
  const Ctl& c = *ctx->h_ctl;
  if (iters) *iters = c.iters;
  if (outcome) *outcome = c.done ? (plss_outcome)c.outcome : PLSS_RUNNING;
  if (hist) for (int k = 0; k <= ctx->maxit; ++k) hist[k] = rec[(size_t)k * REC];
  if (diag) memcpy(diag, rec.data(), 8 * rec.size());
  return PLSS_OK;
}

plss_status plss_solve(plss_ctx* ctx, const double* b, const double* x0, double tol, int32_t tol_mode,
                       int32_t maxit, int32_t flags, double* x, int32_t* iters, double* hist, double* diag,
                       plss_outcome* outcome) {
  NvtxRange nvtx_("plss_solve");
  plss_status s = plss_start(ctx, b, x0, tol, tol_mode, maxit, flags);
  if (s != PLSS_OK) return s;
  cudaStream_t st = ctx->stream;
  // keep <= 2 chunks in flight; poll the device done flag of the older one
  int issued = 0, slot = 0;
  bool pending[2] = {false, false};
  while (issued < maxit) {
    const bool full = (maxit - issued) >= ctx->chunk;
    if (full) {
      NvtxRange chunk_("plss_solve: graph chunk");
      CK(cudaGraphLaunch(ctx->graph_chunk, st));
      issued += ctx->chunk;
    } else {
      for (int i = issued; i < maxit; ++i) CK(cudaGraphLaunch(ctx->graph_one, st));
      issued = maxit;
    }
    CK(cudaMemcpyAsync(&ctx->h_done[slot], &ctx->ctl->done, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(ctx->ev[slot], st));
    pending[slot] = true;
    slot ^= 1;
    if (pending[slot]) {
      const plss_status w = dist_wait(ctx, st, ctx->ev[slot]);
      if (w != PLSS_OK) return w;
      pending[slot] = false;
      if (ctx->h_done[slot]) break;
    }
  }
  return plss_finish(ctx, x, iters, hist, diag, outcome);
}

plss_status plss_spmv(plss_ctx* ctx, const double* x, double* y) {
  NvtxRange nvtx_("plss_spmv");
  if (!ctx || (!x && ctx->n > 0) || (!y && ctx->m > 0)) return PLSS_E_INVALID;
  if (sync_in(ctx) != PLSS_OK) return PLSS_E_CUDA;
  for (int s = 0; s < ctx->S; ++s) {
    SpmvSeg a = ctx->seg1[s];
    a.g = x;
    a.out = y + ctx->R[s];
    a.ctl = nullptr;
    launch_spmv<ROLE_PLAIN>(a, ctx->g1[s], ctx->stream);
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->stream));
  return sync_out(ctx);
}

plss_status plss_spmvT(plss_ctx* ctx, const double* u, double* v) {
  NvtxRange nvtx_("plss_spmvT");
  if (!ctx || (!u && ctx->m > 0) || (!v && ctx->n > 0)) return PLSS_E_INVALID;
  if (sync_in(ctx) != PLSS_OK) return PLSS_E_CUDA;
  // slabs accumulate into the output, whose slices are re-read by TMA: use the (aligned,
  // padded) internal y, then copy out
  double* out = ctx->S > 1 ? ctx->y : v;
  for (int s = 0; s < ctx->S; ++s) {
    SpmvSeg a = ctx->seg2[s];
    a.g = u + (ctx->S > 1 ? ctx->R[s] : 0);
    a.out = out;
    a.ctl = nullptr;
    a.finalize = 0;
    launch_spmv<ROLE_K2>(a, ctx->g2[s], ctx->stream);
  }
  CK(cudaGetLastError());
  if (out != v && ctx->n > 0) CK(cudaMemcpyAsync(v, out, 8 * (size_t)ctx->n, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return sync_out(ctx);
}

plss_status plss_true_residual(plss_ctx* ctx, const double* b, const double* x, double* out) {
  NvtxRange nvtx_("plss_true_residual");
  if (!ctx || !out || (!b && ctx->m > 0) || (!x && ctx->n > 0)) return PLSS_E_INVALID;
  if (sync_in(ctx) != PLSS_OK) return PLSS_E_CUDA;
  cudaStream_t st = ctx->stream;
  const int64_t m = ctx->m, n = ctx->n;
  const int grid = ctx->gnorm;
  double *ax = nullptr, *db = nullptr, *dx = nullptr, *part = nullptr, *res = nullptr;
  unsigned* cnt = nullptr;
  const size_t mb = 8 * (size_t)std::max<int64_t>(m, 1), nb = 8 * (size_t)std::max<int64_t>(n, 1);
  CK(cudaMallocAsync((void**)&ax, mb + 16, st));
  CK(cudaMallocAsync((void**)&part, 16 * (size_t)grid + 16, st));
  CK(cudaMallocAsync((void**)&res, 16, st));
  CK(cudaMallocAsync((void**)&cnt, 16, st));
  CK(cudaMemsetAsync(cnt, 0, 16, st));
  CK(cudaMemsetAsync(res, 0, 16, st));
  const double* bd = b;
  const double* xd = x;
  if (m > 0 && !is_device_ptr(b)) {
    CK(cudaMallocAsync((void**)&db, mb, st));
    CK(cudaMemcpyAsync(db, b, 8 * (size_t)m, cudaMemcpyHostToDevice, st));
    bd = db;
  }
  if (n > 0 && !is_device_ptr(x)) {
    CK(cudaMallocAsync((void**)&dx, nb + 16, st));
    CK(cudaMemcpyAsync(dx, x, 8 * (size_t)n, cudaMemcpyHostToDevice, st));
    xd = dx;
  }
  for (int s = 0; s < ctx->S; ++s) {                 // ax = A x (sequential row sums)
    SpmvSeg a = ctx->seg1[s];
    a.g = xd;
    a.out = ax + ctx->R[s];
    a.ctl = nullptr;
    launch_spmv<ROLE_PLAIN>(a, ctx->g1[s], st);
  }
  if (ctx->cols && m > 0)                    // column blocks: A x = sum over ranks of A_g x_g
    NK(ncclAllReduce(ax, ax, (size_t)m, ncclFloat64, ncclSum, ctx->comm, st));
  if (m > 0) k_true_resid<<<grid, NT, 0, st>>>(bd, ax, m, part, cnt, res);
  CK(cudaGetLastError());
  if (ctx->dist && !ctx->cols) NK(ncclAllReduce(res, res, 2, ncclFloat64, ncclSum, ctx->comm, st));
  double h[2] = {0.0, 0.0};
  CK(cudaMemcpyAsync(h, res, 16, cudaMemcpyDeviceToHost, st));
  for (void* q : {(void*)ax, (void*)db, (void*)dx, (void*)part, (void*)res, (void*)cnt})
    if (q) CK(cudaFreeAsync(q, st));
  CK(cudaStreamSynchronize(st));
  out[0] = std::sqrt(h[0]);
  out[1] = std::sqrt(h[1]);
  return sync_out(ctx);
}

plss_status plss_profile(plss_ctx* ctx, int32_t k, double* ms) {
  NvtxRange nvtx_("plss_profile");
  if (!ctx || !ms || k < 1) return PLSS_E_INVALID;
  if (!ctx->started) { set_err(ctx, "plss_profile before plss_start"); return PLSS_E_STATE; }
  cudaStream_t st = ctx->stream;
  const int nev = 2 * ctx->S + 4;
  std::vector<cudaEvent_t> ev(nev);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  double acc[5] = {0, 0, 0, 0, 0};
  for (int it = 0; it < k && ctx->cols; ++it) {
    // column blocks: K1 | all-reduce of u + rho tail | K2 | dots + all-reduce + phi tail | K3
    const int64_t m = ctx->m;
    double* sc = ctx->scalars + 4;
    CK(cudaEventRecord(ev[0], st));
    for (int s = 0; s < ctx->S; ++s) launch_spmv<ROLE_K1>(ctx->seg1[s], ctx->g1[s], st);
    CK(cudaEventRecord(ev[1], st));
    NK(ncclAllReduce(ctx->r, ctx->r, (size_t)m + 1, ncclFloat64, ncclSum, ctx->comm, st));
    k_rho_tail<<<ctx->gnorm, NT, 0, st>>>(ctx->r, m, ctx->ctl, ctx->rec, ctx->partn, ctx->counters + 3);
    CK(cudaEventRecord(ev[2], st));
    for (int s = 0; s < ctx->S; ++s) launch_spmv<ROLE_K2>(ctx->seg2[s], ctx->g2[s], st);
    CK(cudaEventRecord(ev[3], st));
    k_dots_shard<<<ctx->gdots, NT, 0, st>>>(ctx->y, ctx->p, ctx->n, ctx->ctl, ctx->part2, ctx->counters + 1,
                                            ctx->wi, sc);
    NK(ncclAllReduce(sc + 1, sc + 1, 2, ncclFloat64, ncclSum, ctx->comm, st));
    k_tail_phi<<<1, 1, 0, st>>>(ctx->ctl, ctx->rec, sc);
    CK(cudaEventRecord(ev[4], st));
    k_pxupdate<<<ctx->g3, NT, 0, st>>>(ctx->p, ctx->y, ctx->x, ctx->n, ctx->ctl, ctx->rec, ctx->part3,
                                       ctx->counters + 2, ctx->wi, ctx->r + m);
    if (ctx->rank > 0 && m > 0) CK(cudaMemsetAsync(ctx->r, 0, 8 * (size_t)m, st));
    CK(cudaEventRecord(ev[5], st));
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    const int slot[5] = {0, 2, 1, 3, 4};           // k1, all-reduce + rho tail, k2, dots, k3
    for (int j = 0; j < 5; ++j) {
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, ev[j], ev[j + 1]));
      acc[slot[j]] += t;
    }
  }
  for (int it = 0; it < k && !ctx->cols; ++it) {
    int q = 0;
    CK(cudaEventRecord(ev[q++], st));
    for (int s = 0; s < ctx->S; ++s) {
      launch_spmv<ROLE_K1>(ctx->seg1[s], ctx->g1[s], st);
      CK(cudaEventRecord(ev[q++], st));
      if (ctx->seg2[s].finalize) launch_spmv<ROLE_K2DOTS>(ctx->seg2[s], ctx->g2[s], st);
      else launch_spmv<ROLE_K2>(ctx->seg2[s], ctx->g2[s], st);
      CK(cudaEventRecord(ev[q++], st));
    }
    if (ctx->rsag) {                               // collectives (RS, AR, AG) | shard dots + tail | K3
      double* sc = ctx->scalars + 4;
      NK(ncclReduceScatter(ctx->y, ctx->y + ctx->c0, (size_t)ctx->cnt, ncclFloat64, ncclSum, ctx->comm, st));
      NK(ncclAllReduce(sc, sc, 4, ncclFloat64, ncclSum, ctx->comm, st));
      NK(ncclAllGather(ctx->p + ctx->c0, ctx->p, (size_t)ctx->cnt, ncclFloat64, ctx->comm, st));
      CK(cudaEventRecord(ev[q++], st));
      k_dots_shard<<<ctx->gdots, NT, 0, st>>>(ctx->y + ctx->c0, ctx->p + ctx->c0, ctx->nsh, ctx->ctl, ctx->part2,
                                              ctx->counters + 1, ctx->wi ? ctx->wi + ctx->c0 : nullptr, sc);
      k_tail_rsag<<<1, 1, 0, st>>>(ctx->ctl, ctx->rec, sc);
      CK(cudaEventRecord(ev[q++], st));
      k_pxupdate<<<ctx->g3, NT, 0, st>>>(ctx->p + ctx->c0, ctx->y + ctx->c0, ctx->x + ctx->c0, ctx->nsh, ctx->ctl,
                                         ctx->rec, ctx->part3, ctx->counters + 2,
                                         ctx->wi ? ctx->wi + ctx->c0 : nullptr, sc + 3);
      CK(cudaEventRecord(ev[q++], st));
    } else {
    double* yv = ctx->y;
    if (ctx->dist) {
      if (ctx->peer) {                             // peer reduce of every chunk + wait
        peer_reduce_all(ctx, st);
        k_peer_wait<<<1, 64, 0, st>>>(ctx->ptab, ctx->nranks, peer_nch(ctx), ctx->rank, ctx->ctl);
        yv = ctx->yred;
      } else {
        NK(ncclAllReduce(ctx->y, ctx->y, (size_t)ctx->n + 1, ncclFloat64, ncclSum, ctx->comm, st));
      }
      CK(cudaEventRecord(ev[q++], st));
      k_dots_tail<<<ctx->gdots, NT, 0, st>>>(yv, ctx->p, ctx->n, yv + ctx->n, ctx->ctl, ctx->rec,
                                             ctx->part2, ctx->counters + 1, ctx->wi, ctx->psi_dots);
      CK(cudaEventRecord(ev[q++], st));
    }
    k_pxupdate<<<ctx->g3, NT, 0, st>>>(ctx->p, yv, ctx->x, ctx->n, ctx->ctl, ctx->rec, ctx->part3,
                                       ctx->counters + 2, ctx->wi, nullptr, k3_opts(ctx));
    CK(cudaEventRecord(ev[q++], st));
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    float t;
    int e = 0;
    for (int s = 0; s < ctx->S; ++s) {
      CK(cudaEventElapsedTime(&t, ev[e], ev[e + 1])); acc[0] += t;
      CK(cudaEventElapsedTime(&t, ev[e + 1], ev[e + 2])); acc[1] += t;
      e += 2;
    }
    if (ctx->dist) {
      CK(cudaEventElapsedTime(&t, ev[e], ev[e + 1])); acc[2] += t;
      CK(cudaEventElapsedTime(&t, ev[e + 1], ev[e + 2])); acc[3] += t;
      e += 2;
    }
    CK(cudaEventElapsedTime(&t, ev[e], ev[e + 1])); acc[4] += t;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  for (int i = 0; i < 5; ++i) ms[i] = acc[i] / k;
  return PLSS_OK;
}

plss_status plss_query(const plss_ctx* ctx, int32_t* launches_per_step, int32_t* slabs, int32_t* tile_nnz,
                       int32_t* grid_k1, int32_t* grid_k2, int32_t* sell_segments, int32_t* window_segments) {
  if (!ctx) return PLSS_E_INVALID;
  if (sell_segments) {
    int c = 0;
    for (auto& a : ctx->seg1) c += a.fmt >= 1 && a.fmt <= 3;
    for (auto& a : ctx->seg2) c += a.fmt >= 1 && a.fmt <= 3;
    *sell_segments = c;
  }
  if (window_segments) {
    int c = 0;
    for (auto& a : ctx->seg1) c += a.fmt == 2;
    for (auto& a : ctx->seg2) c += a.fmt == 2;
    *window_segments = c;
  }
  // our kernels per loop step: K1 and K2 per slab (the last K2 as column chunks on a chunked
  // distributed ctx), K3, and the distributed dots / tail kernel
  // (+1 for every globally sorted segment with long rows: k_longrows runs after its slices)
  int extra = 0;
  for (auto& a : ctx->seg1) extra += (a.fmt == 3 && a.nlong > 0 && !a.lin) ? 1 : 0;
  for (auto& a : ctx->seg2) extra += (a.fmt == 3 && a.nlong > 0 && !a.lin) ? 1 : 0;
  if (launches_per_step && ctx->cols)          // K1, K2 per slab; rho tail, dots, phi tail, K3
    *launches_per_step = 2 * ctx->S + 4 + extra;
  else if (launches_per_step)
    *launches_per_step = 2 * ctx->S + 1 + (ctx->dist ? 1 : 0) + (ctx->rsag ? 1 : 0) +
                         (ctx->dch.empty() ? 0 : (int)ctx->dch.size() - 1) +
                         (ctx->peer ? peer_nch(ctx) + 1 : 0) + extra;
  if (slabs) *slabs = ctx->S;
  if (tile_nnz) *tile_nnz = TILE;
  if (grid_k1) *grid_k1 = ctx->g1.empty() ? 0 : ctx->g1[0];
  if (grid_k2) *grid_k2 = ctx->g2.empty() ? 0 : ctx->g2[0];
  return PLSS_OK;
}

plss_status plss_query_segment(const plss_ctx* ctx, int32_t which, int32_t slab, int32_t info[14]) {
  if (!ctx || !info || (which != 1 && which != 2) || slab < 0 || slab >= ctx->S) return PLSS_E_INVALID;
  const SpmvSeg& a = which == 1 ? ctx->seg1[slab] : ctx->seg2[slab];
  info[0] = a.fmt;
  info[1] = a.fmt >= 1 && a.fmt <= 3 && a.perm && !a.gsort ? (a.sig ? a.sig : SIGMA) : 0;
  info[2] = a.gsort;
  info[3] = a.nslices;
  info[4] = a.nlong;
  info[5] = a.stat;
  info[6] = which == 1 ? ctx->g1[slab] : ctx->g2[slab];
  info[7] = a.nrows;
  info[8] = a.lchunk ? a.nchunks : 0;
  info[9] = a.psi3;
  info[10] = ctx->xdefer ? 1 : 0;
  info[11] = a.fmt == 3 && a.gsort && a.s1on ? a.s1beg : -1;
  info[12] = a.fmt == 3 && a.gsort && a.s1on ? a.s1end : -1;
  info[13] = a.fmt == 3 && a.nlong > 0 && a.lin ? 1 : 0;
  return PLSS_OK;
}

plss_status plss_debug_cta_times(plss_ctx* ctx, int32_t which, int32_t slab, uint64_t* out, int32_t* grid) {
  if (!ctx || !out || !grid || (which != 1 && which != 2) || slab < 0 || slab >= ctx->S) return PLSS_E_INVALID;
  const SpmvSeg& a = which == 1 ? ctx->seg1[slab] : ctx->seg2[slab];
  *grid = which == 1 ? ctx->g1[slab] : ctx->g2[slab];
  if (!a.ctat) { set_err(ctx, "create the ctx with PLSS_DBG_CTA=1"); return PLSS_E_STATE; }
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaMemcpy(out, a.ctat, 4 * 8 * (size_t)(*grid), cudaMemcpyDeviceToHost));
  return PLSS_OK;
}

plss_status plss_set_wi(plss_ctx* ctx, const double* wi) {
  NvtxRange nvtx_("plss_set_wi");
  if (!ctx) return PLSS_E_INVALID;
  if (!wi) { ctx->weighted = false; return PLSS_OK; }
  if (sync_in(ctx) != PLSS_OK) return PLSS_E_CUDA;
  cudaStream_t st = ctx->stream;
  const int64_t n = ctx->n;
  if (n > 0) {
    CK(cudaMemcpyAsync(ctx->wi, wi, 8 * (size_t)n, is_device_ptr(wi) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    int* d_err = (int*)(ctx->ws + ctx->L.err);
    CK(cudaMemsetAsync(d_err, 0, 4, st));
    k_check_positive<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ctx->wi, n, d_err);
    CK(cudaGetLastError());
    int h = 0;
    CK(cudaMemcpyAsync(&h, d_err, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h) { set_err(ctx, "WI diagonal entries must be finite and > 0"); return PLSS_E_INVALID; }
  }
  ctx->weighted = true;
  return sync_out(ctx);
}

plss_status plss_column_norms(plss_ctx* ctx, double* c) {
  NvtxRange nvtx_("plss_column_norms");
  if (!ctx || (!c && ctx->n > 0)) return PLSS_E_INVALID;
  if (sync_in(ctx) != PLSS_OK) return PLSS_E_CUDA;
  cudaStream_t st = ctx->stream;
  const int64_t n = ctx->n;
  if (n == 0) return sync_out(ctx);
  // sums of squares into the scan scratch region is too small for n doubles: use y (n+1 doubles),
  // which holds no state between solves
  double* tmp = ctx->y;
  const unsigned g = (unsigned)((n + 255) / 256);
  k_colsq<<<g, 256, 0, st>>>(ctx->A.col_ptr, ctx->A.val_t, n, tmp);
  CK(cudaGetLastError());
  if (ctx->dist && !ctx->cols)              // column blocks hold whole columns
    NK(ncclAllReduce(tmp, tmp, (size_t)n, ncclFloat64, ncclSum, ctx->comm, st));
  k_colnorm_finish<<<g, 256, 0, st>>>(tmp, n);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(c, tmp, 8 * (size_t)n, is_device_ptr(c) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return sync_out(ctx);
}

}  // extern "C"

// ---- shared by the alternative methods (randomized projection, PLSS Kaczmarz) -------------------
// copy out x / iters / history of a run that uses the ctx's x, ctl and rec
static plss_status alt_finish(plss_ctx* ctx, double* x, int32_t* iters, double* hist, double* diag,
                              plss_outcome* outcome) {
  cudaStream_t st = ctx->stream;
  if (x && ctx->n > 0)
    CK(cudaMemcpyAsync(x, ctx->x, 8 * (size_t)ctx->n, is_device_ptr(x) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(ctx->h_ctl, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
  std::vector<double> rec;
  if (hist || diag) {
    rec.resize((size_t)(ctx->maxit + 1) * REC);
    CK(cudaMemcpyAsync(rec.data(), ctx->rec, 8 * rec.size(), cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  if (sync_out(ctx) != PLSS_OK) return PLSS_E_CUDA;
  const Ctl& c = *ctx->h_ctl;
  if (iters) *iters = c.iters;
  if (outcome) *outcome = c.done ? (plss_outcome)c.outcome : (c.iters >= c.maxit ? PLSS_MAXIT : PLSS_RUNNING);
  if (hist) for (int k = 0; k <= ctx->maxit; ++k) hist[k] = rec[(size_t)k * REC];
  if (diag) memcpy(diag, rec.data(), 8 * rec.size());
  return PLSS_OK;
}
// launch up to maxit steps (graphs of ctx->chunk), <= 2 chunks in flight, stop once done
static plss_status alt_run(plss_ctx* ctx, cudaGraphExec_t gchunk, cudaGraphExec_t gone, int maxit) {
  cudaStream_t st = ctx->stream;
  int issued = 0, slot = 0;
  bool pending[2] = {false, false};
  while (issued < maxit) {
    if (maxit - issued >= ctx->chunk) {
      CK(cudaGraphLaunch(gchunk, st));
      issued += ctx->chunk;
    } else {
      for (int i = issued; i < maxit; ++i) CK(cudaGraphLaunch(gone, st));
      issued = maxit;
    }
    CK(cudaMemcpyAsync(&ctx->h_done[slot], &ctx->ctl->done, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(ctx->ev[slot], st));
    pending[slot] = true;
    slot ^= 1;
    if (pending[slot]) {
      CK(cudaEventSynchronize(ctx->ev[slot]));
      pending[slot] = false;
      if (ctx->h_done[slot]) break;
    }
  }
  return PLSS_OK;
}
static plss_status alt_build_graph(plss_ctx* ctx, plss_status (*enqueue)(plss_ctx*), int iters, cudaGraphExec_t* out) {
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  plss_status st = PLSS_OK;
  for (int i = 0; i < iters && st == PLSS_OK; ++i) st = enqueue(ctx);
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
  if (st != PLSS_OK) return st;
  CK(e);
  CK(cudaGraphInstantiate(out, g, 0));
  CK(cudaGraphDestroy(g));
  return PLSS_OK;
}
// common start of an alternative method: control block, history, r = b, x = p = x0 (or 0), ||b||,
// then K1 over the slabs: r_0 = b - A x0, rho_0, record 0 and the stop test
static plss_status alt_start(plss_ctx* ctx, const double* b, const double* x0, double tol, int32_t tol_mode,
                             int32_t maxit) {
  cudaStream_t st = ctx->stream;
  if (sync_in(ctx) != PLSS_OK) return PLSS_E_CUDA;
  const int64_t m = ctx->m, n = ctx->n;
  Ctl& c = *ctx->h_ctl;
  memset(&c, 0, sizeof c);
  c.nbd = 1.0;
  c.tol = tol;
  c.maxit = maxit;
  c.tol_mode = tol_mode;
  c.outcome = OUT_RUNNING;
  CK(cudaMemcpyAsync(ctx->ctl, &c, sizeof(Ctl), cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(ctx->rec, 0, 8 * (size_t)(maxit + 1) * REC, st));
  if (m > 0) CK(cudaMemcpyAsync(ctx->r, b, 8 * (size_t)m, is_device_ptr(b) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  if (n > 0) {
    if (x0) {
      const cudaMemcpyKind kind = is_device_ptr(x0) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
      CK(cudaMemcpyAsync(ctx->p, x0, 8 * (size_t)n, kind, st));   // K1 below gathers x0: r = b - A x0
      CK(cudaMemcpyAsync(ctx->x, x0, 8 * (size_t)n, kind, st));
    } else {
      CK(cudaMemsetAsync(ctx->p, 0, 8 * (size_t)n, st));
      CK(cudaMemsetAsync(ctx->x, 0, 8 * (size_t)n, st));
    }
  }
  k_norm_b<<<ctx->gnorm, NT, 0, st>>>(ctx->r, m, ctx->ctl, ctx->partn, ctx->counters + 3, 1, nullptr);
  for (int s = 0; s < ctx->S; ++s) launch_spmv<ROLE_K1>(ctx->seg1[s], ctx->g1[s], st);
  CK(cudaGetLastError());
  ctx->started = false;          // the PLSS loop state is overwritten
  ctx->rp_started = false;
  ctx->kz_started = false;
  ctx->eg_started = false;
  ctx->maxit = maxit;
  return PLSS_OK;
}

// ---- randomized projection (rp_kernels.cuh) ----------------------------------
static int rp_sms(const plss_ctx* ctx) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->dev);
  return std::max(1, sms);
}
static int rp_ld(int r) { return (r + 7) / 8 * 8; }   // S row stride (floats): whole 32-byte sectors
static void rp_grids(const plss_ctx* ctx, int r, int ld, int* g_gen, int* g_gram) {
  const int sms = rp_sms(ctx);
  const int64_t rows_gen = RP_NT / ((r + 1) / 2), rows_gram = RP_TILE / r;
  (void)ld;
  *g_gen = (int)std::max<int64_t>(1, std::min<int64_t>((ctx->m + rows_gen - 1) / rows_gen, 8 * sms));
  *g_gram = (int)std::max<int64_t>(1, std::min<int64_t>((ctx->n + rows_gram - 1) / rows_gram, 4 * sms));
}
static uint64_t rp_key(uint64_t seed) {   // mix64(seed), host copy of the device finalizer
  uint64_t z = seed;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static size_t rp_bytes(const plss_ctx* ctx, int r) {
  int gg, gm;
  rp_grids(ctx, r, rp_ld(r), &gg, &gm);
  const size_t np = (size_t)r * (r + 1) / 2;
  return align_up(4 * (size_t)ctx->m * rp_ld(r) + 16) + align_up(8 * (size_t)ctx->n * r + 16) +
         align_up(8 * (size_t)gg * r) + align_up(8 * (size_t)gm * np) + align_up(8 * (size_t)RP_RMAX) + align_up(256);
}
static bool rp_valid(const plss_ctx* ctx, int r, double density) {
  return ctx && !ctx->dist && r >= 1 && r <= RP_RMAX && density > 0.0 && density <= 1.0;
}
// carve the caller's workspace; fills everything but ctl / rec / k_fixed / res
static plss_status rp_args(plss_ctx* ctx, int r, uint64_t seed, double density, void* ws, size_t bytes, RpArgs* out) {
  if (!ws || bytes < rp_bytes(ctx, r) || ((uintptr_t)ws % ALIGN) != 0) {
    set_err(ctx, "randomized projection workspace missing, misaligned or smaller than plss_rp_workspace_bytes");
    return PLSS_E_DIM;
  }
  RpArgs a{};
  a.m = ctx->m;
  a.n = ctx->n;
  a.r = r;
  a.h = (r + 1) / 2;
  a.ld = rp_ld(r);
  a.key = rp_key(seed);
  a.density = density;
  rp_grids(ctx, r, a.ld, &a.grid_gen, &a.grid_gram);
  char* w = (char*)ws;
  size_t off = 0;
  auto take = [&](size_t nb) { char* q = w + off; off += align_up(nb); return q; };
  a.S = (float*)take(4 * (size_t)ctx->m * a.ld + 16);
  a.Y = (double*)take(8 * (size_t)ctx->n * r + 16);
  a.vpart = (double*)take(8 * (size_t)a.grid_gen * r);
  a.mpart = (double*)take(8 * (size_t)a.grid_gram * r * (r + 1) / 2);
  a.z = (double*)take(8 * (size_t)RP_RMAX);
  a.colctr = (unsigned*)take(256);
  a.pol_stream = ctx->seg1.empty() ? 0ull : ctx->seg1[0].pol_first;
  a.p = ctx->p;
  a.x = ctx->x;
  a.col_ptr = ctx->A.col_ptr;
  a.row_idx = ctx->A.row_idx;
  a.val_t = ctx->A.val_t;
  *out = a;
  return PLSS_OK;
}
static void rp_launch_spmm(const RpArgs& a, int grid, cudaStream_t st) {
  if (a.r <= 8) k_rp_spmm<8, 1><<<grid, RP_NT, 0, st>>>(a);
  else if (a.r <= 16) k_rp_spmm<16, 1><<<grid, RP_NT, 0, st>>>(a);
  else if (a.r <= 32) k_rp_spmm<32, 1><<<grid, RP_NT, 0, st>>>(a);
  else k_rp_spmm<32, 2><<<grid, RP_NT, 0, st>>>(a);
}
// one resident wave: the kernel takes columns from a global counter
static int rp_spmm_grid(const plss_ctx* ctx, int r, int ld) {
  int occ = 1;
  (void)ld;
  const void* fn = r <= 8 ? (const void*)k_rp_spmm<8, 1> : r <= 16 ? (const void*)k_rp_spmm<16, 1>
                 : r <= 32 ? (const void*)k_rp_spmm<32, 1> : (const void*)k_rp_spmm<32, 2>;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, RP_NT, 0) != cudaSuccess || occ < 1) occ = 1;
  int g = 8;                                        // lanes per column
  while (g < r && g < 32) g <<= 1;
  const int cpw = 32 / g;                           // columns per warp
  const int64_t cols_per_cta = (int64_t)(RP_NT / 32) * cpw;
  return (int)std::max<int64_t>(1, std::min<int64_t>((ctx->n + cols_per_cta - 1) / cols_per_cta, (int64_t)occ * rp_sms(ctx)));
}
static plss_status rp_enqueue_step(plss_ctx* ctx) {
  cudaStream_t st = ctx->stream;
  const RpArgs& a = ctx->rp;
  k_rp_gen<<<a.grid_gen, RP_NT, 0, st>>>(a);
  rp_launch_spmm(a, ctx->rp_gspmm, st);
  k_rp_gram<<<a.grid_gram, RP_NT, 0, st>>>(a);
  k_rp_solve<<<1, RP_NT, 0, st>>>(a);
  k_rp_update<<<ctx->rp_gupd, RP_NT, 0, st>>>(a);
  for (int s = 0; s < ctx->S; ++s) launch_spmv<ROLE_K1>(ctx->seg1[s], ctx->g1[s], st);
  CK(cudaGetLastError());
  return PLSS_OK;
}

extern "C" {

size_t plss_rp_workspace_bytes(const plss_ctx* ctx, int32_t r) {
  if (!rp_valid(ctx, r, 1.0)) return 0;
  return rp_bytes(ctx, r);
}

plss_status plss_rp_start(plss_ctx* ctx, int32_t r, uint64_t seed, double density, void* workspace,
                          size_t ws_bytes, const double* b, const double* x0, double tol, int32_t tol_mode,
                          int32_t maxit) {
  NvtxRange nvtx_("plss_rp_start");
  if (!ctx) return PLSS_E_INVALID;
  if (!rp_valid(ctx, r, density) || !(tol >= 0.0) || maxit < 1 || maxit > ctx->L.maxit_cap ||
      (tol_mode != 0 && tol_mode != 1)) {
    set_err(ctx, ctx->dist ? "randomized projection runs on a single-device ctx"
                           : "invalid r (1..64) / density (0, 1] / tol / tol_mode / maxit");
    return PLSS_E_INVALID;
  }
  if (!b && ctx->m > 0) { set_err(ctx, "b is NULL"); return PLSS_E_INVALID; }
  RpArgs a;
  plss_status ps = rp_args(ctx, r, seed, density, workspace, ws_bytes, &a);
  if (ps != PLSS_OK) return ps;
  a.res = ctx->r;
  a.ctl = ctx->ctl;
  a.rec = ctx->rec;
  a.k_fixed = 0;
  if ((ps = alt_start(ctx, b, x0, tol, tol_mode, maxit)) != PLSS_OK) return ps;
  const int64_t n = ctx->n;
  ctx->rp = a;
  ctx->rp_gspmm = rp_spmm_grid(ctx, r, rp_ld(r));
  ctx->rp_gupd = (int)std::max<int64_t>(1, std::min<int64_t>((n + RP_NT - 1) / RP_NT, 8 * (int64_t)rp_sms(ctx)));
  if (ctx->rp_graph_chunk) { CK(cudaGraphExecDestroy(ctx->rp_graph_chunk)); ctx->rp_graph_chunk = nullptr; }
  if (ctx->rp_graph_one) { CK(cudaGraphExecDestroy(ctx->rp_graph_one)); ctx->rp_graph_one = nullptr; }
  if ((ps = alt_build_graph(ctx, rp_enqueue_step, ctx->chunk, &ctx->rp_graph_chunk)) != PLSS_OK) return ps;
  if ((ps = alt_build_graph(ctx, rp_enqueue_step, 1, &ctx->rp_graph_one)) != PLSS_OK) return ps;
  ctx->rp_started = true;
  return PLSS_OK;
}

plss_status plss_rp_step(plss_ctx* ctx, int32_t k) {
  NvtxRange nvtx_("plss_rp_step");
  if (!ctx) return PLSS_E_INVALID;
  if (!ctx->rp_started) { set_err(ctx, "plss_rp_step before plss_rp_start"); return PLSS_E_STATE; }
  if (k < 0) return PLSS_E_INVALID;
  for (int i = 0; i + ctx->chunk <= k; i += ctx->chunk) CK(cudaGraphLaunch(ctx->rp_graph_chunk, ctx->stream));
  for (int i = 0; i < k % ctx->chunk; ++i) CK(cudaGraphLaunch(ctx->rp_graph_one, ctx->stream));
  return PLSS_OK;
}

plss_status plss_rp_finish(plss_ctx* ctx, double* x, int32_t* iters, double* hist, double* diag,
                           plss_outcome* outcome) {
  NvtxRange nvtx_("plss_rp_finish");
  if (!ctx) return PLSS_E_INVALID;
  if (!ctx->rp_started) { set_err(ctx, "plss_rp_finish before plss_rp_start"); return PLSS_E_STATE; }
  return alt_finish(ctx, x, iters, hist, diag, outcome);
}

plss_status plss_rp_solve(plss_ctx* ctx, int32_t r, uint64_t seed, double density, void* workspace,
                          size_t ws_bytes, const double* b, const double* x0, double tol, int32_t tol_mode,
                          int32_t maxit, double* x, int32_t* iters, double* hist, double* diag,
                          plss_outcome* outcome) {
  NvtxRange nvtx_("plss_rp_solve");
  plss_status s = plss_rp_start(ctx, r, seed, density, workspace, ws_bytes, b, x0, tol, tol_mode, maxit);
  if (s != PLSS_OK) return s;
  if ((s = alt_run(ctx, ctx->rp_graph_chunk, ctx->rp_graph_one, maxit)) != PLSS_OK) return s;
  return plss_rp_finish(ctx, x, iters, hist, diag, outcome);
}

plss_status plss_rp_profile(plss_ctx* ctx, int32_t k, double* ms) {
  if (!ctx || !ms || k < 1) return PLSS_E_INVALID;
  if (!ctx->rp_started) { set_err(ctx, "plss_rp_profile before plss_rp_start"); return PLSS_E_STATE; }
  cudaStream_t st = ctx->stream;
  const RpArgs& a = ctx->rp;
  constexpr int NK = 6;
  cudaEvent_t ev[NK + 1];
  for (auto& e : ev) CK(cudaEventCreate(&e));
  double acc[NK] = {0, 0, 0, 0, 0, 0};
  for (int it = 0; it < k; ++it) {
    CK(cudaEventRecord(ev[0], st));
    k_rp_gen<<<a.grid_gen, RP_NT, 0, st>>>(a);
    CK(cudaEventRecord(ev[1], st));
    rp_launch_spmm(a, ctx->rp_gspmm, st);
    CK(cudaEventRecord(ev[2], st));
    k_rp_gram<<<a.grid_gram, RP_NT, 0, st>>>(a);
    CK(cudaEventRecord(ev[3], st));
    k_rp_solve<<<1, RP_NT, 0, st>>>(a);
    CK(cudaEventRecord(ev[4], st));
    k_rp_update<<<ctx->rp_gupd, RP_NT, 0, st>>>(a);
    CK(cudaEventRecord(ev[5], st));
    for (int s = 0; s < ctx->S; ++s) launch_spmv<ROLE_K1>(ctx->seg1[s], ctx->g1[s], st);
    CK(cudaEventRecord(ev[6], st));
    CK(cudaGetLastError());
    CK(cudaEventSynchronize(ev[6]));
    for (int j = 0; j < NK; ++j) {
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, ev[j], ev[j + 1]));
      acc[j] += t;
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  for (int j = 0; j < NK; ++j) ms[j] = acc[j] / k;
  return PLSS_OK;
}

plss_status plss_rp_sketch(plss_ctx* ctx, int32_t r, uint64_t seed, double density, int32_t k, int32_t ld,
                           float* S) {
  if (!ctx || !rp_valid(ctx, r, density) || k < 1 || ld < r || (ld & 1) || ld > 2 * RP_NT || (!S && ctx->m > 0))
    return PLSS_E_INVALID;
  RpArgs a{};
  a.m = ctx->m;
  a.n = ctx->n;
  a.r = r;
  a.h = (r + 1) / 2;
  a.ld = ld;
  a.key = rp_key(seed);
  a.density = density;
  a.S = S;
  a.k_fixed = k;
  int gm;
  rp_grids(ctx, r, ld, &a.grid_gen, &gm);
  if (sync_in(ctx) != PLSS_OK) return PLSS_E_CUDA;
  k_rp_gen<<<a.grid_gen, RP_NT, 0, ctx->stream>>>(a);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->stream));
  return sync_out(ctx);
}

plss_status plss_spmmT(plss_ctx* ctx, int32_t r, int32_t ld, const float* S, double* Y) {
  if (!ctx || r < 1 || r > RP_RMAX || ld < r || (!S && ctx->m > 0) || (!Y && ctx->n > 0)) return PLSS_E_INVALID;
  RpArgs a{};
  a.m = ctx->m;
  a.n = ctx->n;
  a.r = r;
  a.ld = ld;
  a.S = const_cast<float*>(S);
  a.Y = Y;
  a.col_ptr = ctx->A.col_ptr;
  a.row_idx = ctx->A.row_idx;
  a.val_t = ctx->A.val_t;
  a.pol_stream = ctx->seg1.empty() ? 0ull : ctx->seg1[0].pol_first;
  if (sync_in(ctx) != PLSS_OK) return PLSS_E_CUDA;
  CK(cudaMallocAsync((void**)&a.colctr, sizeof(unsigned), ctx->stream));
  CK(cudaMemsetAsync(a.colctr, 0, sizeof(unsigned), ctx->stream));
  rp_launch_spmm(a, rp_spmm_grid(ctx, r, ld), ctx->stream);
  CK(cudaGetLastError());
  CK(cudaFreeAsync(a.colctr, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return sync_out(ctx);
}

}  // extern "C"

// ---- PLSS Kaczmarz (kz_kernels.cuh) ------------------------------------------
static void kz_grids(const plss_ctx* ctx, int* g_gemv, int* g_res) {
  const int sms = rp_sms(ctx);
  *g_gemv = (int)std::max<int64_t>(1, std::min<int64_t>((ctx->n + KZ_TL - 1) / KZ_TL, 8 * (int64_t)sms));
  *g_res = (int)std::max<int64_t>(1, std::min<int64_t>((ctx->m + KZ_NT - 1) / KZ_NT, 4 * (int64_t)sms));
}
static size_t kz_bytes(const plss_ctx* ctx, int kmax) {
  int gg, gr;
  kz_grids(ctx, &gg, &gr);
  const size_t m = (size_t)ctx->m, n = (size_t)ctx->n, K = (size_t)kmax;
  return align_up(8 * n * K) + align_up(8 * m * K) + 2 * align_up(8 * K) + 2 * align_up(8 * n) + align_up(8 * m) +
         align_up(8 * (size_t)gg) + align_up(16 * (size_t)gr) + align_up(256) + align_up(sizeof(KzState)) +
         align_up(4 * (size_t)(ctx->L.maxit_cap + 1));
}
static plss_status kz_enqueue_step(plss_ctx* ctx) {
  cudaStream_t st = ctx->stream;
  const KzArgs& a = ctx->kz;
  k_kz_gemv<<<a.grid_gemv, KZ_NT, 0, st>>>(a);
  if (a.fused) {
    k_kz_resid<true><<<a.grid_res, KZ_NT, 0, st>>>(a);
  } else {
    for (int s = 0; s < ctx->S; ++s) launch_spmv<ROLE_PLAIN>(ctx->kz_seg[s], ctx->g1[s], st);
    k_kz_resid<false><<<a.grid_res, KZ_NT, 0, st>>>(a);
  }
  CK(cudaGetLastError());
  return PLSS_OK;
}

extern "C" {

size_t plss_kz_workspace_bytes(const plss_ctx* ctx, int32_t kmax) {
  if (!ctx || ctx->dist || kmax < 1) return 0;
  return kz_bytes(ctx, kmax);
}

plss_status plss_kz_start(plss_ctx* ctx, int32_t kmax, void* workspace, size_t ws_bytes, const int32_t* rows,
                          const double* b, const double* x0, double tol, int32_t tol_mode, int32_t maxit) {
  NvtxRange nvtx_("plss_kz_start");
  if (!ctx) return PLSS_E_INVALID;
  if (ctx->dist || kmax < 1 || !(tol >= 0.0) || maxit < 1 || maxit > ctx->L.maxit_cap ||
      (tol_mode != 0 && tol_mode != 1) || !rows) {
    set_err(ctx, ctx->dist ? "PLSS Kaczmarz runs on a single-device ctx"
                           : "invalid kmax / tol / tol_mode / maxit, or rows is NULL");
    return PLSS_E_INVALID;
  }
  if (!b && ctx->m > 0) { set_err(ctx, "b is NULL"); return PLSS_E_INVALID; }
  if (!workspace || ws_bytes < kz_bytes(ctx, kmax) || ((uintptr_t)workspace % ALIGN) != 0) {
    set_err(ctx, "PLSS Kaczmarz workspace missing, misaligned or smaller than plss_kz_workspace_bytes");
    return PLSS_E_DIM;
  }
  cudaStream_t st = ctx->stream;
  std::vector<int32_t> hrows((size_t)maxit);
  CK(cudaMemcpyAsync(hrows.data(), rows, 4 * (size_t)maxit, is_device_ptr(rows) ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int32_t i : hrows)
    if (i < 0 || i >= ctx->m) { set_err(ctx, "row index out of range in the Kaczmarz row schedule"); return PLSS_E_INVALID; }
  KzArgs a{};
  a.m = ctx->m;
  a.n = ctx->n;
  a.kmax = kmax;
  a.row_ptr = ctx->A.row_ptr;
  a.col_idx = ctx->A.col_idx;
  a.val = ctx->A.val;
  kz_grids(ctx, &a.grid_gemv, &a.grid_res);
  char* w = (char*)workspace;
  size_t off = 0;
  auto take = [&](size_t nb) { char* q = w + off; off += align_up(nb); return q; };
  const size_t m = (size_t)ctx->m, n = (size_t)ctx->n, K = (size_t)kmax;
  a.P = (double*)take(8 * n * K);
  a.AP = (double*)take(8 * m * K);
  a.theta = (double*)take(8 * K);
  a.w = (double*)take(8 * K);
  a.arow = (double*)take(8 * n);
  a.pk = (double*)take(8 * n);
  a.apk = (double*)take(8 * m);
  a.part_th = (double*)take(8 * (size_t)a.grid_gemv);
  a.part_rho = (double*)take(16 * (size_t)a.grid_res);
  a.counter = (unsigned*)take(256);
  a.st = (KzState*)take(sizeof(KzState));
  int32_t* drows = (int32_t*)take(4 * (size_t)(ctx->L.maxit_cap + 1));
  a.rows = drows;
  a.r = ctx->r;
  a.x = ctx->x;
  a.ctl = ctx->ctl;
  a.rec = ctx->rec;
  plss_status ps = alt_start(ctx, b, x0, tol, tol_mode, maxit);
  if (ps != PLSS_OK) return ps;
  KzState s0{};
  s0.prev_row = -1;
  CK(cudaMemcpyAsync(drows, hrows.data(), 4 * (size_t)maxit, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(a.st, &s0, sizeof s0, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(a.counter, 0, 256, st));
  if (n > 0) CK(cudaMemsetAsync(a.arow, 0, 8 * n, st));
  CK(cudaStreamSynchronize(st));   // hrows / s0 are host temporaries
  {                                                  // short rows only: fuse (A p)_l into k_kz_resid
    int32_t* dmax = nullptr;
    int32_t hmax = 0;
    CK(cudaMallocAsync((void**)&dmax, sizeof(int32_t), st));
    CK(cudaMemsetAsync(dmax, 0, sizeof(int32_t), st));
    if (m > 0) k_max_row_len<<<(unsigned)std::min<int64_t>((m + 255) / 256, 4096), 256, 0, st>>>(a.row_ptr, (long long)m, dmax);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&hmax, dmax, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(dmax, st));
    CK(cudaStreamSynchronize(st));
    a.fused = (hmax <= KZ_FUSE_MAXROW && env_int("PLSS_KZ_FUSE", 1) != 0) ? 1 : 0;
  }
  ctx->kz = a;
  k_kz_prep<<<1, KZ_NT, 0, st>>>(a);   // the first step's row; later steps' rows are prepared by k_kz_resid
  CK(cudaGetLastError());
  ctx->kz_seg = ctx->seg1;
  for (int s = 0; s < ctx->S; ++s) {
    SpmvSeg& g = ctx->kz_seg[s];
    g.g = a.pk;
    g.out = a.apk + ctx->R[s];
    g.ctl = ctx->ctl;                // no-op once done
  }
  if (ctx->kz_graph_chunk) { CK(cudaGraphExecDestroy(ctx->kz_graph_chunk)); ctx->kz_graph_chunk = nullptr; }
  if (ctx->kz_graph_one) { CK(cudaGraphExecDestroy(ctx->kz_graph_one)); ctx->kz_graph_one = nullptr; }
  if ((ps = alt_build_graph(ctx, kz_enqueue_step, ctx->chunk, &ctx->kz_graph_chunk)) != PLSS_OK) return ps;
  if ((ps = alt_build_graph(ctx, kz_enqueue_step, 1, &ctx->kz_graph_one)) != PLSS_OK) return ps;
  ctx->kz_started = true;
  return PLSS_OK;
}

plss_status plss_kz_step(plss_ctx* ctx, int32_t k) {
  NvtxRange nvtx_("plss_kz_step");
  if (!ctx) return PLSS_E_INVALID;
  if (!ctx->kz_started) { set_err(ctx, "plss_kz_step before plss_kz_start"); return PLSS_E_STATE; }
  if (k < 0) return PLSS_E_INVALID;
  for (int i = 0; i + ctx->chunk <= k; i += ctx->chunk) CK(cudaGraphLaunch(ctx->kz_graph_chunk, ctx->stream));
  for (int i = 0; i < k % ctx->chunk; ++i) CK(cudaGraphLaunch(ctx->kz_graph_one, ctx->stream));
  return PLSS_OK;
}

plss_status plss_kz_finish(plss_ctx* ctx, double* x, int32_t* iters, double* hist, double* diag,
                           plss_outcome* outcome) {
  NvtxRange nvtx_("plss_kz_finish");
  if (!ctx) return PLSS_E_INVALID;
  if (!ctx->kz_started) { set_err(ctx, "plss_kz_finish before plss_kz_start"); return PLSS_E_STATE; }
  return alt_finish(ctx, x, iters, hist, diag, outcome);
}

plss_status plss_kz_solve(plss_ctx* ctx, int32_t kmax, void* workspace, size_t ws_bytes, const int32_t* rows,
                          const double* b, const double* x0, double tol, int32_t tol_mode, int32_t maxit, double* x,
                          int32_t* iters, double* hist, double* diag, plss_outcome* outcome) {
  NvtxRange nvtx_("plss_kz_solve");
  plss_status s = plss_kz_start(ctx, kmax, workspace, ws_bytes, rows, b, x0, tol, tol_mode, maxit);
  if (s != PLSS_OK) return s;
  if ((s = alt_run(ctx, ctx->kz_graph_chunk, ctx->kz_graph_one, maxit)) != PLSS_OK) return s;
  return plss_kz_finish(ctx, x, iters, hist, diag, outcome);
}

plss_status plss_kz_profile(plss_ctx* ctx, int32_t k, double* ms) {
  if (!ctx || !ms || k < 1) return PLSS_E_INVALID;
  if (!ctx->kz_started) { set_err(ctx, "plss_kz_profile before plss_kz_start"); return PLSS_E_STATE; }
  cudaStream_t st = ctx->stream;
  const KzArgs& a = ctx->kz;
  constexpr int NK = 4;
  cudaEvent_t ev[NK + 1];
  for (auto& e : ev) CK(cudaEventCreate(&e));
  double acc[NK] = {0, 0, 0, 0};
  for (int it = 0; it < k; ++it) {
    CK(cudaEventRecord(ev[0], st));
    CK(cudaEventRecord(ev[1], st));     // row preparation is fused into k_kz_resid (slot 0 stays ~0)
    k_kz_gemv<<<a.grid_gemv, KZ_NT, 0, st>>>(a);
    CK(cudaEventRecord(ev[2], st));
    if (!a.fused)
      for (int s = 0; s < ctx->S; ++s) launch_spmv<ROLE_PLAIN>(ctx->kz_seg[s], ctx->g1[s], st);
    CK(cudaEventRecord(ev[3], st));
    if (a.fused) k_kz_resid<true><<<a.grid_res, KZ_NT, 0, st>>>(a);
    else k_kz_resid<false><<<a.grid_res, KZ_NT, 0, st>>>(a);
    CK(cudaEventRecord(ev[4], st));
    CK(cudaGetLastError());
    CK(cudaEventSynchronize(ev[4]));
    for (int j = 0; j < NK; ++j) {
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, ev[j], ev[j + 1]));
      acc[j] += t;
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  for (int j = 0; j < NK; ++j) ms[j] = acc[j] / k;
  return PLSS_OK;
}

}  // extern "C"

// ---- growing-sketch engine, triangular factorization (eg_kernels.cuh) --------
static void eg_grids(const plss_ctx* ctx, int* g_t, int* g_s, int* g_g) {
  const int sms = rp_sms(ctx);
  *g_t = (int)std::max<int64_t>(1, (ctx->n + EG_RT_SMALL - 1) / EG_RT_SMALL);   // max row ranges of Y^T y
  *g_s = (int)std::max<int64_t>(1, std::min<int64_t>((ctx->m + EG_NT - 1) / EG_NT, 4 * (int64_t)sms));
  *g_g = (int)std::max<int64_t>(1, std::min<int64_t>((ctx->n + 63) / 64, 8 * (int64_t)sms));
}
static size_t eg_bytes(const plss_ctx* ctx, int kmax) {
  int gt, gs, gg;
  eg_grids(ctx, &gt, &gs, &gg);
  const size_t m = (size_t)ctx->m, n = (size_t)ctx->n, K = (size_t)kmax;
  return align_up(8 * n * K) + align_up(8 * K * K) + 6 * align_up(8 * (K + 2)) + align_up(16 * (K / 32 + 1)) + align_up(256) +
         align_up(8 * n) + align_up(16 * (size_t)gg) + align_up(256) + align_up(8 * (K + 1) * (size_t)gt) +
         align_up(8 * (size_t)gs) + align_up(8 * m) + align_up(sizeof(EgState)) + align_up(4 * (size_t)(ctx->L.maxit_cap + 1));
}
static void eg_enqueue_sketch(plss_ctx* ctx, cudaStream_t st) {
  const EgArgs& a = ctx->eg;
  if (a.mode == EG_IDENTITY) {
    k_eg_row<<<1, EG_NT, 0, st>>>(a);
  } else {
    if (a.mode == EG_GAUSSIAN) k_eg_gauss<<<a.grid_s, EG_NT, 0, st>>>(a);
    for (int s = 0; s < ctx->S; ++s) launch_spmv<ROLE_K2>(ctx->eg_seg[s], ctx->g2[s], st);   // y = A^T s
  }
}
// the factorization part of a step (between the sketch and K1); `ev` (optional) receives events
// after the Y^T y reduction and after the triangular / reflector work (plss_eg_profile)
static void eg_enqueue_factor(plss_ctx* ctx, cudaStream_t st, cudaEvent_t ev_a, cudaEvent_t ev_b) {
  const EgArgs& a = ctx->eg;
  const int gred = (a.kmax + 2 + EG_NT / 32 - 1) / (EG_NT / 32);
  const int gy = (a.kmax + EG_CT - 1) / EG_CT;
  const dim3 gT((unsigned)std::max<int64_t>(1, (a.n + EG_RT - 1) / EG_RT), gy), gTs((unsigned)a.grid_t, gy);
  k_eg_gemvT<0, EG_RT><<<gT, EG_NT, 0, st>>>(a);
  k_eg_gemvT<0, EG_RT_SMALL><<<gTs, EG_NT, 0, st>>>(a);
  k_eg_red<0><<<gred, EG_NT, 0, st>>>(a);
  if (ev_a) cudaEventRecord(ev_a, st);
  if (a.factor == 0) {
    k_eg_triu<<<gred, EG_NT, 0, st>>>(a);
    k_eg_trit<<<a.grid_tri, EG_NT, 0, st>>>(a);
    if (ev_b) cudaEventRecord(ev_b, st);
    k_eg_gemv<0><<<a.grid_g, EG_NT, 0, st>>>(a);
  } else {
    k_qr_b<<<gred, EG_NT, 0, st>>>(a);
    k_qr_w<<<a.grid_g, EG_NT, 0, st>>>(a);
    k_qr_v<<<a.grid_s, EG_NT, 0, st>>>(a);
    k_eg_gemvT<1, EG_RT><<<gT, EG_NT, 0, st>>>(a);
    k_eg_gemvT<1, EG_RT_SMALL><<<gTs, EG_NT, 0, st>>>(a);
    k_eg_red<1><<<gred, EG_NT, 0, st>>>(a);
    k_qr_tri<<<a.grid_tri, EG_NT, 0, st>>>(a);
    if (ev_b) cudaEventRecord(ev_b, st);
    k_eg_gemv<1><<<a.grid_g, EG_NT, 0, st>>>(a);
  }
}
static plss_status eg_enqueue_step(plss_ctx* ctx) {
  cudaStream_t st = ctx->stream;
  eg_enqueue_sketch(ctx, st);
  eg_enqueue_factor(ctx, st, nullptr, nullptr);
  for (int s = 0; s < ctx->S; ++s) launch_spmv<ROLE_K1>(ctx->seg1[s], ctx->g1[s], st);     // r -= A p, rho, stop
  CK(cudaGetLastError());
  return PLSS_OK;
}

extern "C" {

size_t plss_eg_workspace_bytes(const plss_ctx* ctx, int32_t kmax) {
  if (!ctx || ctx->dist || kmax < 1) return 0;
  return eg_bytes(ctx, kmax);
}

plss_status plss_eg_start(plss_ctx* ctx, int32_t sketch, int32_t factor, int32_t kmax, void* workspace,
                          size_t ws_bytes, const int32_t* rows, uint64_t seed, const double* b, const double* x0,
                          double tol, int32_t tol_mode, int32_t maxit) {
  NvtxRange nvtx_("plss_eg_start");
  if (!ctx) return PLSS_E_INVALID;
  if (ctx->dist || kmax < 1 || sketch < EG_RESIDUAL || sketch > EG_GAUSSIAN || (factor != 0 && factor != 1) ||
      !(tol >= 0.0) || maxit < 1 ||
      maxit > ctx->L.maxit_cap || (tol_mode != 0 && tol_mode != 1) || (sketch == EG_IDENTITY && !rows)) {
    set_err(ctx, ctx->dist ? "the growing-sketch engine runs on a single-device ctx"
                           : "invalid sketch / kmax / tol / tol_mode / maxit, or rows is NULL for identity sketches");
    return PLSS_E_INVALID;
  }
  if (!b && ctx->m > 0) { set_err(ctx, "b is NULL"); return PLSS_E_INVALID; }
  if (!workspace || ws_bytes < eg_bytes(ctx, kmax) || ((uintptr_t)workspace % ALIGN) != 0) {
    set_err(ctx, "engine workspace missing, misaligned or smaller than plss_eg_workspace_bytes");
    return PLSS_E_DIM;
  }
  cudaStream_t st = ctx->stream;
  std::vector<int32_t> hrows;
  if (sketch == EG_IDENTITY) {
    hrows.resize((size_t)maxit);
    CK(cudaMemcpyAsync(hrows.data(), rows, 4 * (size_t)maxit, is_device_ptr(rows) ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int32_t i : hrows)
      if (i < 0 || i >= ctx->m) { set_err(ctx, "row index out of range in the identity sketch"); return PLSS_E_INVALID; }
  }
  EgArgs a{};
  a.m = ctx->m;
  a.n = ctx->n;
  a.kmax = kmax;
  a.mode = sketch;
  a.factor = factor;
  a.row_ptr = ctx->A.row_ptr;
  a.col_idx = ctx->A.col_idx;
  a.val = ctx->A.val;
  a.key = rp_key(seed);
  eg_grids(ctx, &a.grid_t, &a.grid_s, &a.grid_g);
  char* w = (char*)workspace;
  size_t off = 0;
  auto take = [&](size_t nb) { char* q = w + off; off += align_up(nb); return q; };
  const size_t m = (size_t)ctx->m, n = (size_t)ctx->n, K = (size_t)kmax;
  a.Y = (double*)take(8 * n * K);
  a.R = (double*)take(8 * K * K);
  a.dinv = (double*)take(8 * (K + 2));
  a.gv = (double*)take(8 * (K + 2));
  a.th = (double*)take(8 * (K + 2));
  a.uv = (double*)take(8 * (K + 2));
  a.grid_tri = (int)(K / 32 + 1);
  a.part_tri = (double*)take(16 * (K / 32 + 1));
  a.counter = (unsigned*)take(256);
  a.cv = (double*)take(8 * (K + 2));
  a.zv = (double*)take(8 * (K + 2));
  a.w = (double*)take(8 * n);
  a.part_w = (double*)take(16 * (size_t)a.grid_g);
  a.counter2 = (unsigned*)take(256);
  a.part = (double*)take(8 * (K + 1) * (size_t)a.grid_t);
  a.part_rs = (double*)take(8 * (size_t)a.grid_s);
  a.s = (double*)take(8 * m);
  a.st = (EgState*)take(sizeof(EgState));
  int32_t* drows = (int32_t*)take(4 * (size_t)(ctx->L.maxit_cap + 1));
  a.rows = drows;
  a.y = ctx->y;
  a.p = ctx->p;
  a.x = ctx->x;
  a.r = ctx->r;
  a.ctl = ctx->ctl;
  a.rec = ctx->rec;
  plss_status ps = alt_start(ctx, b, x0, tol, tol_mode, maxit);
  if (ps != PLSS_OK) return ps;
  EgState s0{};
  s0.prev_row = -1;
  CK(cudaMemcpyAsync(a.st, &s0, sizeof s0, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(a.counter, 0, 256, st));
  CK(cudaMemsetAsync(a.counter2, 0, 256, st));
  if (!hrows.empty()) CK(cudaMemcpyAsync(drows, hrows.data(), 4 * (size_t)maxit, cudaMemcpyHostToDevice, st));
  if (n > 0) CK(cudaMemsetAsync(ctx->y, 0, 8 * n, st));
  CK(cudaStreamSynchronize(st));   // host temporaries
  ctx->eg = a;
  ctx->eg_seg = ctx->seg2;
  for (int s = 0; s < ctx->S; ++s) {
    SpmvSeg& g = ctx->eg_seg[s];
    const double* src = sketch == EG_GAUSSIAN ? a.s : ctx->r;
    g.g = src + (ctx->S > 1 ? ctx->R[s] : 0);
    g.out = ctx->y;
    g.finalize = 0;
    g.ctl = ctx->ctl;
  }
  if (ctx->eg_graph_chunk) { CK(cudaGraphExecDestroy(ctx->eg_graph_chunk)); ctx->eg_graph_chunk = nullptr; }
  if (ctx->eg_graph_one) { CK(cudaGraphExecDestroy(ctx->eg_graph_one)); ctx->eg_graph_one = nullptr; }
  if ((ps = alt_build_graph(ctx, eg_enqueue_step, ctx->chunk, &ctx->eg_graph_chunk)) != PLSS_OK) return ps;
  if ((ps = alt_build_graph(ctx, eg_enqueue_step, 1, &ctx->eg_graph_one)) != PLSS_OK) return ps;
  ctx->eg_started = true;
  return PLSS_OK;
}

plss_status plss_eg_step(plss_ctx* ctx, int32_t k) {
  NvtxRange nvtx_("plss_eg_step");
  if (!ctx) return PLSS_E_INVALID;
  if (!ctx->eg_started) { set_err(ctx, "plss_eg_step before plss_eg_start"); return PLSS_E_STATE; }
  if (k < 0) return PLSS_E_INVALID;
  for (int i = 0; i + ctx->chunk <= k; i += ctx->chunk) CK(cudaGraphLaunch(ctx->eg_graph_chunk, ctx->stream));
  for (int i = 0; i < k % ctx->chunk; ++i) CK(cudaGraphLaunch(ctx->eg_graph_one, ctx->stream));
  return PLSS_OK;
}

plss_status plss_eg_finish(plss_ctx* ctx, double* x, int32_t* iters, double* hist, double* diag,
                           plss_outcome* outcome) {
  NvtxRange nvtx_("plss_eg_finish");
  if (!ctx) return PLSS_E_INVALID;
  if (!ctx->eg_started) { set_err(ctx, "plss_eg_finish before plss_eg_start"); return PLSS_E_STATE; }
  return alt_finish(ctx, x, iters, hist, diag, outcome);
}

plss_status plss_eg_solve(plss_ctx* ctx, int32_t sketch, int32_t factor, int32_t kmax, void* workspace,
                          size_t ws_bytes, const int32_t* rows, uint64_t seed, const double* b, const double* x0,
                          double tol, int32_t tol_mode, int32_t maxit, double* x, int32_t* iters, double* hist,
                          double* diag, plss_outcome* outcome) {
  NvtxRange nvtx_("plss_eg_solve");
  plss_status s = plss_eg_start(ctx, sketch, factor, kmax, workspace, ws_bytes, rows, seed, b, x0, tol, tol_mode, maxit);
  if (s != PLSS_OK) return s;
  if ((s = alt_run(ctx, ctx->eg_graph_chunk, ctx->eg_graph_one, maxit)) != PLSS_OK) return s;
  return plss_eg_finish(ctx, x, iters, hist, diag, outcome);
}

plss_status plss_eg_profile(plss_ctx* ctx, int32_t k, double* ms) {
  if (!ctx || !ms || k < 1) return PLSS_E_INVALID;
  if (!ctx->eg_started) { set_err(ctx, "plss_eg_profile before plss_eg_start"); return PLSS_E_STATE; }
  cudaStream_t st = ctx->stream;
  constexpr int NK = 5;
  cudaEvent_t ev[NK + 1];
  for (auto& e : ev) CK(cudaEventCreate(&e));
  double acc[NK] = {0, 0, 0, 0, 0};
  for (int it = 0; it < k; ++it) {
    CK(cudaEventRecord(ev[0], st));
    eg_enqueue_sketch(ctx, st);
    CK(cudaEventRecord(ev[1], st));
    eg_enqueue_factor(ctx, st, ev[2], ev[3]);
    CK(cudaEventRecord(ev[4], st));
    for (int s = 0; s < ctx->S; ++s) launch_spmv<ROLE_K1>(ctx->seg1[s], ctx->g1[s], st);
    CK(cudaEventRecord(ev[5], st));
    CK(cudaGetLastError());
    CK(cudaEventSynchronize(ev[5]));
    for (int j = 0; j < NK; ++j) {
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, ev[j], ev[j + 1]));
      acc[j] += t;
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  for (int j = 0; j < NK; ++j) ms[j] = acc[j] / k;
  return PLSS_OK;
}

}  // extern "C"

extern "C" {

void plss_destroy(plss_ctx* ctx) {
  if (!ctx) return;
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->graph_chunk) cudaGraphExecDestroy(ctx->graph_chunk);
  if (ctx->graph_one) cudaGraphExecDestroy(ctx->graph_one);
  if (ctx->rp_graph_chunk) cudaGraphExecDestroy(ctx->rp_graph_chunk);
  if (ctx->rp_graph_one) cudaGraphExecDestroy(ctx->rp_graph_one);
  if (ctx->kz_graph_chunk) cudaGraphExecDestroy(ctx->kz_graph_chunk);
  if (ctx->kz_graph_one) cudaGraphExecDestroy(ctx->kz_graph_one);
  if (ctx->eg_graph_chunk) cudaGraphExecDestroy(ctx->eg_graph_chunk);
  if (ctx->eg_graph_one) cudaGraphExecDestroy(ctx->eg_graph_one);
  for (void* q : ctx->ipc_open) cudaIpcCloseMemHandle(q);
  if (ctx->sym) cudaFree(ctx->sym);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  for (void* q : ctx->dbg_bufs) cudaFree(q);
  for (void* q : ctx->chunk_bufs) cudaFree(q);
  if (ctx->slabmajor) cudaFree(ctx->slabmajor);
  if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
  if (ctx->join_ev) cudaEventDestroy(ctx->join_ev);
  if (ctx->fork_stream) cudaStreamDestroy(ctx->fork_stream);
  for (auto& e : ctx->ev_ch) if (e) cudaEventDestroy(e);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  if (ctx->h_done) cudaFreeHost(ctx->h_done);
  if (ctx->h_ctl) cudaFreeHost(ctx->h_ctl);
  for (auto& e : ctx->ev) if (e) cudaEventDestroy(e);
  if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
  if (ctx->ev_out) cudaEventDestroy(ctx->ev_out);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* plss_status_str(plss_status s) {
  switch (s) {
    case PLSS_OK: return "ok";
    case PLSS_E_INVALID: return "invalid argument";
    case PLSS_E_DIM: return "dimension mismatch";
    case PLSS_E_FORMAT: return "matrix format violation";
    case PLSS_E_CUDA: return "CUDA error";
    case PLSS_E_NCCL: return "NCCL error";
    case PLSS_E_NOMEM: return "out of host memory";
    case PLSS_E_STATE: return "call out of order";
  }
  return "unknown status";
}

const char* plss_last_error(const plss_ctx* ctx) {
  if (ctx) return ctx->err.c_str();
  return g_last_error.c_str();
}

}  // extern "C"

extern "C" {

// test entry point: one step of the peer-memory all-reduce over G virtual ranks on this device
// (peer_kernels.cuh: the kernels of the distributed step, launched cooperatively with one grid row
// per virtual rank, since their CTAs wait on one another)
plss_status plss_peer_reduce_emulate(int32_t G, double* const* part, double* const* red, uint32_t* const* flags,
                                     int32_t nch, const int64_t* bounds, void* cuda_stream) {
  if (G < 1 || G > PEER_MAX || nch < 1 || nch > PEER_NCH || !part || !red || !flags || !bounds) {
    g_last_error = "invalid argument";
    return PLSS_E_INVALID;
  }
  for (int c = 0; c < nch; ++c)
    if (bounds[c] < 0 || bounds[c + 1] < bounds[c]) { g_last_error = "bounds must be non-decreasing"; return PLSS_E_INVALID; }
  PeerTab t{};
  for (int h = 0; h < G; ++h) {
    if (!part[h] || !red[h] || !flags[h]) { g_last_error = "NULL buffer"; return PLSS_E_INVALID; }
    t.part[h] = part[h];
    t.red[h] = red[h];
    t.flg[h] = flags[h];
  }
  int dev = 0, sms = 1, occ = 1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_peer_reduce, PEER_NT, 0);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  int gx = std::max(1, std::min(16, occ * sms / G));
  int zero = 0;
  const Ctl* noctl = nullptr;
  for (int c = 0; c < nch && e == cudaSuccess; ++c) {
    long long lo = bounds[c], hi = bounds[c + 1];
    void* args[] = {&t, &G, &zero, &c, &lo, &hi, &noctl};
    e = cudaLaunchCooperativeKernel((const void*)k_peer_reduce, dim3(gx, G), dim3(PEER_NT), args, 0, s);
  }
  if (e == cudaSuccess) {
    void* args[] = {&t, &G, &nch, &zero, &noctl};
    e = cudaLaunchCooperativeKernel((const void*)k_peer_wait, dim3(1, G), dim3(64), args, 0, s);
  }
  unsigned err = 0;
  for (int h = 0; h < G && e == cudaSuccess; ++h) {
    unsigned v = 0;
    e = cudaMemcpyAsync(&v, flags[h] + PF_ERR, sizeof v, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    err |= v;
  }
  if (e != cudaSuccess) { g_last_error = cudaGetErrorString(e); return PLSS_E_CUDA; }
  if (err) { g_last_error = "peer-memory step: a virtual rank did not arrive within 20 s"; return PLSS_E_CUDA; }
  return PLSS_OK;
}

}  // extern "C"
