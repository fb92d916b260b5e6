// Microbenchmark: can the TMA unit gather faster than the LSU path on B200?
// Random 8-byte gathers from a 64 MB fp64 vector (L2-resident), three ways:
//   ldg     : one ld.global.nc per gather (the SpMV kernels' path; ~1 gather/clk/SM measured)
//   gather4 : cp.async.bulk.tensor.2d.tile::gather4 of 4 random 16-byte rows (the fp64 pair that
//             holds each wanted element) into shared memory, mbarrier completion, then LDS
//   lds     : random 8-byte loads from a 128 KB shared-memory array (the window kernel's path)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather4_bench gather4_bench.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CKR(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(256) k_ldg(const int32_t* __restrict__ idx, const double* __restrict__ x, long long n,
                                             double* out) {
  double s = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n; i += 8 * stride) {
    int c[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) c[u] = __ldcs(idx + i + u * stride);
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(x + c[u]);
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  if (s == 1234.5) out[0] = s;
}

// Each thread issues K gather4 ops (4K gathers) per round into its own 128-byte slots (the TMA
// destination must be 128-byte aligned; 64 bytes are used); one
// mbarrier per stage counts all threads' bytes; NS stages in flight.
template <int K, int NS>
__global__ void __launch_bounds__(128) k_g4(const __grid_constant__ CUtensorMap tm, const int32_t* __restrict__ idx,
                                            long long n, double* out) {
  extern __shared__ __align__(128) unsigned char buf[];
  __shared__ uint64_t bar[NS];
  const int t = threadIdx.x;
  if (t == 0) {
    for (int q = 0; q < NS; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(&bar[q])), "r"((unsigned)blockDim.x) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long per_round = (long long)blockDim.x * K * 4;
  const long long rounds_total = n / per_round;
  double s = 0.0;
  auto issue = [&](long long r, int q) {
    const int32_t* ip = idx + r * per_round + (long long)t * K * 4;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[q])), "r"((unsigned)(K * 64))
                 : "memory");
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int4 c = *reinterpret_cast<const int4*>(ip + 4 * k);
      unsigned char* dst = buf + ((size_t)q * blockDim.x * K + (size_t)t * K + k) * 128;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
          ::"r"(s32(dst)), "l"(&tm), "r"(0), "r"(c.x >> 1), "r"(c.y >> 1), "r"(c.z >> 1), "r"(c.w >> 1),
          "r"(s32(&bar[q]))
          : "memory");
    }
  };
  long long r = blockIdx.x;
  const long long G = gridDim.x;
  for (int q = 0; q < NS && r + q * G < rounds_total; ++q) issue(r + q * G, q);
  int j = 0;
  for (; r < rounds_total; r += G, ++j) {
    const int q = j % NS;
    const unsigned par = (unsigned)(j / NS) & 1u;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                   : "=r"(ok) : "r"(s32(&bar[q])), "r"(par) : "memory");
    const int32_t* ip = idx + r * per_round + (long long)t * K * 4;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int4 c = *reinterpret_cast<const int4*>(ip + 4 * k);
      const double* row = reinterpret_cast<const double*>(buf + ((size_t)q * blockDim.x * K + (size_t)t * K + k) * 128);
      s += row[0 + (c.x & 1)] + row[2 + (c.y & 1)] + row[4 + (c.z & 1)] + row[6 + (c.w & 1)];
    }
    __syncthreads();
    if (r + NS * G < rounds_total) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(r + NS * G, q);
    }
  }
  if (s == 1234.5) out[0] = s;
}

__global__ void __launch_bounds__(256) k_lds(const int32_t* __restrict__ idx, long long n, double* out, int mask) {
  extern __shared__ double sb[];
  for (int i = threadIdx.x; i <= mask; i += blockDim.x) sb[i] = i;
  __syncthreads();
  double s = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n; i += 8 * stride) {
    int c[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) c[u] = __ldcs(idx + i + u * stride) & mask;
#pragma unroll
    for (int u = 0; u < 8; ++u) s += sb[c[u]];
  }
  if (s == 1234.5) out[0] = s;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  int sms;
  CKR(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int clk_khz;
  CKR(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  const long long ng = 256ll << 20;            // gathers
  const long long xs = 8ll << 20;              // 8M doubles = 64 MB
  int32_t* idx;
  double *x, *out;
  CKR(cudaMalloc(&idx, ng * 4));
  CKR(cudaMalloc(&x, xs * 8));
  CKR(cudaMalloc(&out, 64));
  CKR(cudaMemset(x, 0, xs * 8));
  std::vector<int32_t> h(ng);
  srand(7);
  for (long long i = 0; i < ng; ++i) h[i] = (int32_t)(((long long)rand() * 2654435761ll) % xs);
  CKR(cudaMemcpy(idx, h.data(), ng * 4, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto&& launch) {
    launch();
    CKR(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) launch();
    cudaEventRecord(e1);
    CKR(cudaEventSynchronize(e1));
    CKR(cudaGetLastError());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double gps = 3.0 * ng / (ms / 1e3);
    printf("%-28s %7.1f Ggather/s = %.3f gathers/clk/SM @%.3f GHz (base clock attr)\n", name, gps / 1e9,
           gps / (sms * clk_khz * 1e3), clk_khz / 1e6);
  };
  timeit("ldg 16 CTA/SM x 256", [&] { k_ldg<<<sms * 16, 256>>>(idx, x, ng, out); });
  CKR(cudaFuncSetAttribute(k_lds, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024));
  timeit("lds 128KB, 1 CTA/SM x 256", [&] { k_lds<<<sms, 256, 128 * 1024>>>(idx, ng, out, 16384 - 1); });
  timeit("lds 32KB, 6 CTA/SM x 256", [&] { k_lds<<<sms * 6, 256, 32 * 1024>>>(idx, ng, out, 4096 - 1); });

  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  CKR(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
  EncodeFn enc = (EncodeFn)fn;
  CUtensorMap tm;
  cuuint64_t gdim[2] = {2, (cuuint64_t)(xs / 2)};
  cuuint64_t gstr[1] = {16};
  cuuint32_t box[2] = {2, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, gdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode box {2,1}: %d\n", (int)cr);
  if (cr != CUDA_SUCCESS) return 0;
  auto run_g4 = [&](auto kern, int K, int NS, int ctas_per_sm, const char* name) {
    const size_t smem = (size_t)NS * 128 * K * 128;
    CKR(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    timeit(name, [&] { kern<<<sms * ctas_per_sm, 128, smem>>>(tm, idx, ng, out); });
  };
  run_g4(k_g4<2, 2>, 2, 2, 4, "gather4 K2 NS2 4 CTA/SM");
  run_g4(k_g4<4, 2>, 4, 2, 4, "gather4 K4 NS2 4 CTA/SM");
  run_g4(k_g4<4, 3>, 4, 3, 2, "gather4 K4 NS3 2 CTA/SM");
  run_g4(k_g4<8, 2>, 8, 2, 2, "gather4 K8 NS2 2 CTA/SM");
  return 0;
}
