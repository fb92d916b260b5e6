/* examples/solve.c -- the C ABI (include/plss.h) without Python: build a small consistent system,
 * copy its CSR + CSC arrays to the device, solve with PLSS, print the iteration count and residual.
 *
 *   gcc -std=c99 -O2 -I include examples/solve.c -o solve \
 *       -L paper_2207_07615_b200 -lplss -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2207_07615_b200
 *   ./solve
 *
 * A = tridiag(-1, 4, -1) of size N (square, well conditioned), x* = 1, b = A x*. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "plss.h"

#define N 1000
#define CHECK(call)                                                                      \
  do {                                                                                   \
    plss_status s_ = (call);                                                             \
    if (s_ != PLSS_OK) {                                                                 \
      fprintf(stderr, "%s: %s (%s)\n", #call, plss_status_str(s_), plss_last_error(NULL)); \
      return 1;                                                                          \
    }                                                                                    \
  } while (0)

static void* to_device(const void* h, size_t bytes) {
  void* d = NULL;
  /* 16-byte padded allocations (plss.h conventions) */
  if (cudaMalloc(&d, (bytes + 15) / 16 * 16 + 16) != cudaSuccess) return NULL;
  cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice);
  return d;
}

int main(void) {
  int32_t row_ptr[N + 1], col_idx[3 * N];
  double val[3 * N], b[N], x[N], hist[101];
  int64_t nnz = 0;
  for (int i = 0; i < N; ++i) {
    row_ptr[i] = (int32_t)nnz;
    for (int j = i - 1; j <= i + 1; ++j) {
      if (j < 0 || j >= N) continue;
      col_idx[nnz] = j;
      val[nnz] = (j == i) ? 4.0 : -1.0;
      ++nnz;
    }
    b[i] = (i == 0 || i == N - 1) ? 3.0 : 2.0;    /* A * ones */
  }
  row_ptr[N] = (int32_t)nnz;
  /* A is symmetric, so its CSC copy has the same arrays */
  plss_matrix A;
  memset(&A, 0, sizeof A);
  A.m = N;
  A.n = N;
  A.nnz = nnz;
  A.row_ptr = to_device(row_ptr, sizeof row_ptr);
  A.col_idx = to_device(col_idx, 4 * (size_t)nnz);
  A.val = to_device(val, 8 * (size_t)nnz);
  A.col_ptr = A.row_ptr;
  A.row_idx = A.col_idx;
  A.val_t = A.val;
  A.validate = 1;
  if (!A.row_ptr || !A.col_idx || !A.val) { fprintf(stderr, "no CUDA device\n"); return 1; }
  plss_options opt = {0, 0, 100, 0};
  size_t ws_bytes = plss_workspace_bytes(&A, &opt);
  void* ws = NULL;
  if (ws_bytes == 0 || cudaMalloc(&ws, ws_bytes) != cudaSuccess) { fprintf(stderr, "workspace\n"); return 1; }
  plss_ctx* ctx = NULL;
  CHECK(plss_create(&A, &opt, ws, ws_bytes, NULL, &ctx));
  int32_t iters = 0;
  plss_outcome outcome;
  CHECK(plss_solve(ctx, b, NULL, 1e-12, 0, 100, 0, x, &iters, hist, NULL, &outcome));
  double err = 0.0;
  for (int i = 0; i < N; ++i) err = (x[i] - 1.0) * (x[i] - 1.0) > err ? (x[i] - 1.0) * (x[i] - 1.0) : err;
  printf("PLSS: %d iterations, outcome %d, final relative residual %.3e, max |x - 1|^2 %.3e\n", iters,
         (int)outcome, hist[iters < 100 ? iters : 99], err);
  plss_destroy(ctx);
  cudaFree(ws);
  return outcome == PLSS_CONVERGED ? 0 : 2;
}
