// Microbenchmark: random 8-byte gather throughput on B200 (the inner operation of K1 / K2).
// Streams an index array (coalesced) and gathers x[idx] with different load flavours and
// index locality, to find the per-SM L1TEX wavefront ceiling that bounds the SpMV kernels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

template <int MODE>
__device__ __forceinline__ double ld(const double* p) {
  double v;
  if (MODE == 0) v = *p;                                                     // ld.global (L1 allocate)
  else if (MODE == 1) v = __ldg(p);                                          // ld.global.nc
  else if (MODE == 2) asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));   // L2 only
  else asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(256) gather(const int32_t* __restrict__ idx, const double* __restrict__ x,
                                              long long n, double* out) {
  double s = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n; i += 8 * stride) {
    int c[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) c[u] = __ldcs(idx + i + u * stride);
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = ld<MODE>(x + c[u]);
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; i < n; i += stride) s += ld<MODE>(x + idx[i]);
  if (s == 1234.5) out[0] = s;
}

__global__ void stream_copy(const double* a, double* b, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    b[i] = a[i];
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long ngather = 256ll << 20;  // 256M gathers
  int32_t* idx;
  double *x, *out, *big;
  cudaMalloc(&idx, ngather * 4);
  cudaMalloc(&out, 64);
  const long long xmax = 64ll << 20;      // up to 64M doubles (512 MB)
  cudaMalloc(&x, xmax * 8);
  cudaMemset(x, 0, xmax * 8);
  cudaMalloc(&big, 2ll << 30);
  std::vector<int32_t> h(ngather);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // HBM copy reference
  {
    long long nn = (1ll << 30) / 8;
    stream_copy<<<sms * 8, 256>>>(big, big + nn, nn);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) stream_copy<<<sms * 8, 256>>>(big, big + nn, nn);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy: %.1f GB/s\n", 5.0 * 2 * nn * 8 / (ms / 1e3) / 1e9);
  }
  const long long sizes[3] = {8ll << 20, 8ll << 20, 64ll << 20};  // 64 MB random, 64 MB banded, 512 MB random
  const char* names[3] = {"64MB random", "64MB banded(+-1024 sorted per 12)", "512MB random"};
  for (int cfg = 0; cfg < 3; ++cfg) {
    const long long xs = sizes[cfg];
    srand(1234);
    for (long long i = 0; i < ngather; ++i) {
      if (cfg == 1) {
        long long row = i / 12;
        long long c = (row * 8) % xs;  // like C5's band: column ~ row*n/m with n/m = 1/8 -> use row/8
        c = (row / 8) % xs;
        long long lo = std::max(0ll, std::min(c - 1024, xs - 2049));
        h[i] = (int32_t)(lo + (rand() % 2049));
      } else {
        h[i] = (int32_t)(((long long)rand() * 2654435761ll) % xs);
      }
    }
    cudaMemcpy(idx, h.data(), ngather * 4, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 4; ++mode) {
      for (int occ : {8, 16}) {
        auto run = [&]() {
          if (mode == 0) gather<0><<<sms * occ, 256>>>(idx, x, ngather, out);
          if (mode == 1) gather<1><<<sms * occ, 256>>>(idx, x, ngather, out);
          if (mode == 2) gather<2><<<sms * occ, 256>>>(idx, x, ngather, out);
          if (mode == 3) gather<3><<<sms * occ, 256>>>(idx, x, ngather, out);
        };
        run();
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) run();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double gps = 3.0 * ngather / (ms / 1e3);
        printf("%-36s mode %d grid %2dx: %7.1f Ggather/s  = %.3f gathers/clk/SM @1.965GHz\n", names[cfg], mode, occ,
               gps / 1e9, gps / (sms * 1.965e9));
      }
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(err));
  return 0;
}
