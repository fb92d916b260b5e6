// Microbenchmark: throughput of uniformly random 8-byte gathers that should hit L2, as a function
// of the gathered vector's size, alone and next to a coalesced read stream (K1's mix: 12 stream
// bytes per entry, half of the entries gathering a uniform column). Indices come from a 32-bit LCG
// in registers (no index stream), so only the gathers (and the optional stream) touch memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_l2_bench gather_l2_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ double ld_first(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_na(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// STREAM: 0 none, 1 a read stream of SB doubles per gather (plain), 2 the same with L2 evict-first
template <int STREAM, int U>
__global__ void __launch_bounds__(1024, 1) gath(const double* __restrict__ p, unsigned mask, const double* __restrict__ s,
                                                long long per_thread, double* out) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, nt = (long long)gridDim.x * blockDim.x;
  unsigned x = (unsigned)tid * 2654435761u + 12345u;
  double acc = 0.0;
  for (long long k = 0; k < per_thread; k += U) {
    double sv[U];
    if (STREAM) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double* q = s + ((k + u) * nt + tid);   // coalesced across the grid, 8 B per gather
        sv[u] = STREAM == 2 ? ld_first(q, pol) : ld_na(q);
      }
    }
    double g[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      x = x * 1664525u + 1013904223u;
      g[u] = __ldg(p + ((x >> 7) & mask));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += g[u] + (STREAM ? sv[u] : 0.0);
  }
  if (acc == 1234.5) out[0] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double *p, *s, *out;
  const long long pmax = 1ll << 25;          // 32M doubles = 256 MB
  CK(cudaMalloc(&p, pmax * 8));
  CK(cudaMemset(p, 0, pmax * 8));
  const long long nt = (long long)sms * 1024, per = 512;
  CK(cudaMalloc(&s, nt * per * 8));          // 512 doubles per thread: 620 MB stream
  CK(cudaMemset(s, 0, nt * per * 8));
  CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](auto kern, unsigned mask, const char* nm) {
    kern<<<sms, 1024>>>(p, mask, s, per, out);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) kern<<<sms, 1024>>>(p, mask, s, per, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    const double g = (double)nt * per;
    printf("%-44s vec %4lld MB: %.3f ms  %6.1f Ggather/s = %.3f /clk/SM  sectors %5.2f TB/s\n", nm,
           (long long)(mask + 1ll) * 8 >> 20, ms, g / ms / 1e6, g / (ms * 1e-3) / sms / (clk * 1e3),
           g * 32 / (ms * 1e-3) / 1e12);
  };
  for (unsigned lg : {17u, 20u, 21u, 22u, 23u, 24u, 25u}) {
    const unsigned mask = (1u << lg) - 1;
    run(gath<0, 8>, mask, "gathers only (U 8)");
    run(gath<1, 8>, mask, "gathers + 8 B/gather stream (U 8)");
    run(gath<2, 8>, mask, "gathers + 8 B/gather stream evict-first (U 8)");
  }
  return 0;
}
