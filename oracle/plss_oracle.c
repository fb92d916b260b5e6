/*
 * PLSS CPU ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously correct binary64 implementation of Algorithm 1 (PLSS) of
 * arXiv 2207.07615 with WI = I, or a diagonal WI = B^T B given as a vector
 * (PLSS W, L714-765 / L777-783), used only by tests/, bench.py's cpu_baseline /
 * reference arm and __graft_entry__.smoke() to check the CUDA path. It shares no code, header,
 * table or constant generator with paper_2207_07615_b200/ and must never be linked into it.
 *
 * Compile: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC (oracle/__init__.py).
 * All sums are sequential in ascending index order, no FMA contraction, no compensated summation
 * ("All arithmetic in binary64; no extended-precision accumulation").
 *
 * Threads (oracle_set_threads, default 1 = the sequential oracle): with T > 1 the row / column
 * loops and the element-wise updates are split statically over T threads -- every output element
 * is still one sequential ascending sum computed by one thread, so A x, A^T u and every vector
 * update are bitwise those of T = 1 -- and a dot product is T fixed blocks [len t/T, len (t+1)/T),
 * each summed sequentially, then the T partials summed in block order: deterministic for a given T,
 * a different (equally valid) summation order than T = 1. Used for the full-size parity tests and
 * the host-core baseline (SURVEY 8(d) oracle_omp); pinned against T = 1 in tests/test_oracle_pins.py.
 *
 * Readings of the paper used here (listed in DESIGN.md "Readings"):
 *  R1  gamma = (theta/rho)*beta as in Algorithm 1 line "gamma_k=(theta_k/rho_k)*beta_k"
 *      (Thm 4.1 proof L698/L704), NOT the misprinted theorem form L639-643.
 *  R2  stop test right after rho is recomputed (after L804), <= comparison (L977, L992),
 *      iters = number of updates applied to x, init update counts as 1; maxit caps iters.
 *  R3  ||r0|| = 0 -> converged with 0 iterations; relative mode with ||b|| = 0 uses denominator 1.
 *  R4  stop on the recursive residual r <- r - A p (L801), as Algorithm 1 does.
 *  R5  breakdown guards phi <= 1e-300 (Y_VANISHED) and tau - 1 <= 1e-14 (STAGNATION)
 *      (SPEC.md L147, L156); freeze mode for fixed-iteration timing: once hist <= FREEZE_H or a
 *      guard fires (or tol is met), beta = gamma = 0 for the rest of the run.
 *  R7  psi = y_k^T p_{k-1} is a diagnostic only (identity psi = -rho).
 *  R8  tau = sqrt(theta*phi)/rho; beta = 1/((tau-1)*(tau+1)) in exactly Algorithm 1's order.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int g_threads = 1;

/* Number of host threads of the oracle (1: sequential). */
void oracle_set_threads(int t) { g_threads = t < 1 ? 1 : t; }
int oracle_get_threads(void) { return g_threads; }

#define OR_CONVERGED 0
#define OR_MAXIT 1
#define OR_Y_VANISHED 2
#define OR_STAGNATION 3

/* Per-iteration record, 8 doubles: hist, rho, phi, psi, theta, tau, beta, gamma. */
#define REC 8

/* Column norms c_j = ||A_{:,j}|| (sum of squares in ascending row order, then sqrt); zero columns
 * get 1. PLSS W takes WI = diag(c), i.e. W = diag(1/||A_{:,j}||) (PAPER.md L761-764,
 * L977-979). */
void oracle_column_norms(int64_t n, const int32_t *col_ptr, const double *val_t, double *c) {
    for (int64_t j = 0; j < n; ++j) {
        double s = 0.0;
        for (int64_t k = col_ptr[j]; k < col_ptr[j + 1]; ++k) s = s + val_t[k] * val_t[k];
        c[j] = s > 0.0 ? sqrt(s) : 1.0;
    }
}

/* y = A x over CSR: y_i = sum_j a_ij x_j in ascending j ("matvec"). */
void oracle_spmv(int64_t m, const int32_t *row_ptr, const int32_t *col_idx, const double *val,
                 const double *x, double *y) {
    #pragma omp parallel for num_threads(g_threads) schedule(static) if (g_threads > 1)
    for (int64_t i = 0; i < m; ++i) {
        double s = 0.0;
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) s = s + val[k] * x[col_idx[k]];
        y[i] = s;
    }
}

/* v = A^T u over the CSC copy: v_j = sum_i a_ij u_i in ascending i. */
void oracle_spmvT(int64_t n, const int32_t *col_ptr, const int32_t *row_idx, const double *val_t,
                  const double *u, double *v) {
    #pragma omp parallel for num_threads(g_threads) schedule(static) if (g_threads > 1)
    for (int64_t j = 0; j < n; ++j) {
        double s = 0.0;
        for (int64_t k = col_ptr[j]; k < col_ptr[j + 1]; ++k) s = s + val_t[k] * u[row_idx[k]];
        v[j] = s;
    }
}

/* sum_i a_i b_i (b = NULL: a_i wi_i a_i with wi = w, or a_i a_i) over [lo, hi), ascending */
static double dot_range(int64_t lo, int64_t hi, const double *a, const double *b, const double *w) {
    double s = 0.0;
    for (int64_t i = lo; i < hi; ++i) s = s + a[i] * (b ? b[i] : (w ? w[i] * a[i] : a[i]));
    return s;
}

/* T = 1: one sequential sum. T > 1: T fixed blocks summed in block order (see the header). */
static double dot_blocks(int64_t len, const double *a, const double *b, const double *w) {
    const int T = g_threads;
    if (T <= 1) return dot_range(0, len, a, b, w);
    double *part = (double *)malloc(sizeof(double) * (size_t)T);
    #pragma omp parallel for num_threads(T) schedule(static, 1)
    for (int t = 0; t < T; ++t) part[t] = dot_range(len * t / T, len * (t + 1) / T, a, b, w);
    double s = 0.0;
    for (int t = 0; t < T; ++t) s = s + part[t];
    free(part);
    return s;
}

static double dot(int64_t len, const double *a, const double *b) { return dot_blocks(len, a, b, NULL); }

/* theta = p^T (WI p) with WI = diag(wi), or p^T p when wi is NULL (Alg. 1) */
static double wdot(int64_t len, const double *p, const double *wi) { return dot_blocks(len, p, NULL, wi); }

/*
 * Algorithm 1, following SURVEY.md 8(c)'s transcription. wi (nullable, n):
 * the diagonal of WI; NULL is WI = I. WIy = WI \ y = y ./ wi (L788, L805, applied element-wise as
 * the paper does for diagonal WI, L819-821).
 * x0 may be NULL (zero). x (n) receives the final iterate. rec (nullable) receives
 * (maxit+1)*REC doubles: rec[k*REC + 0..7] = hist_k, rho_k, phi, psi, theta, tau, beta, gamma
 * where at k the values are those computed in loop step k (k = 0: initialization).
 * freeze != 0: fixed-iteration mode (R5). Returns outcome; *iters_out = updates applied.
 * P_out (nullable, maxit*n doubles) receives the updates p_1 .. p_iters (test pins only).
 */
int oracle_plss(int64_t m, int64_t n,
                const int32_t *row_ptr, const int32_t *col_idx, const double *val,
                const int32_t *col_ptr, const int32_t *row_idx, const double *val_t,
                const double *b, const double *x0, const double *wi, double tol, int tol_mode,
                int32_t maxit, int freeze, double freeze_h,
                double *x, int32_t *iters_out, double *rec, double *P_out) {
    double *r = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    double *y = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double *wy = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double *p = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double *Ap = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    int outcome = OR_MAXIT, frozen = 0, stopped = 0;
    int32_t iters = 0;
    if (rec) memset(rec, 0, sizeof(double) * (size_t)(maxit + 1) * REC);

    /* nb = ||b||, denominator of the relative stop test (R3) */
    double nb = sqrt(dot(m, b, b));
    double nbd = (tol_mode == 0 && nb > 0.0) ? nb : 1.0;

    /* x = x0; r = b - A x0  (Alg. 1) */
    for (int64_t j = 0; j < n; ++j) x[j] = x0 ? x0[j] : 0.0;
    for (int64_t i = 0; i < m; ++i) r[i] = b[i];
    if (x0) {
        oracle_spmv(m, row_ptr, col_idx, val, x0, Ap);
        for (int64_t i = 0; i < m; ++i) r[i] = r[i] - Ap[i];
    }
    /* rho = r^T r; stop test before initialization (R2/R3) */
    double rho = dot(m, r, r);
    double h = sqrt(rho) / nbd;
    if (rec) { rec[0] = h; rec[1] = rho; }
    if (rho == 0.0 || h <= tol) {
        if (!freeze) { outcome = OR_CONVERGED; goto done; }
        frozen = 1; outcome = OR_CONVERGED; stopped = 1;
    } else if (freeze && h <= freeze_h) {
        frozen = 1;
    }

    /* y = A^T r; WIy = WI \ y; phi = y^T WIy; p = (rho/phi) WIy; theta = p^T (WI p); x = x + p
     * (L786-797) */
    oracle_spmvT(n, col_ptr, row_idx, val_t, r, y);
    for (int64_t j = 0; j < n; ++j) wy[j] = wi ? y[j] / wi[j] : y[j];
    double phi = dot(n, y, wy);
    double gamma0 = 0.0;
    if (phi <= 1e-300) {
        if (!freeze) { outcome = OR_Y_VANISHED; goto done; }
        if (!stopped) { outcome = OR_Y_VANISHED; stopped = 1; }
        frozen = 1;
    }
    if (!frozen) gamma0 = rho / phi;
    for (int64_t j = 0; j < n; ++j) p[j] = gamma0 * wy[j];
    double theta = wdot(n, p, wi);
    for (int64_t j = 0; j < n; ++j) x[j] = x[j] + p[j];
    iters = 1;
    if (P_out) for (int64_t j = 0; j < n; ++j) P_out[j] = p[j];
    if (rec) { rec[2] = phi; rec[4] = theta; rec[7] = gamma0; }

    while (iters < maxit) {                                     /* L799 */
        double *rk = rec ? rec + (size_t)iters * REC : NULL;
        /* r = r - A p  (L801, eq:recRes) */
        oracle_spmv(m, row_ptr, col_idx, val, p, Ap);
        #pragma omp parallel for num_threads(g_threads) schedule(static) if (g_threads > 1)
        for (int64_t i = 0; i < m; ++i) r[i] = r[i] - Ap[i];
        rho = dot(m, r, r);                                     /* L804 */
        h = sqrt(rho) / nbd;
        if (rk) { rk[0] = h; rk[1] = rho; }
        if (h <= tol) {                                         /* stop test (R2) */
            if (!freeze) { outcome = OR_CONVERGED; goto done; }
            if (!stopped) { outcome = OR_CONVERGED; stopped = 1; }
            frozen = 1;
        } else if (freeze && h <= freeze_h) {
            frozen = 1;
        }
        /* y = A^T r; WIy = WI \ y; phi = y^T WIy; psi = y^T p_{k-1}  (L802, L805-806; L671-672) */
        oracle_spmvT(n, col_ptr, row_idx, val_t, r, y);
        #pragma omp parallel for num_threads(g_threads) schedule(static) if (g_threads > 1)
        for (int64_t j = 0; j < n; ++j) wy[j] = wi ? y[j] / wi[j] : y[j];
        phi = dot(n, y, wy);
        double psi = dot(n, y, p);
        double tau = 0.0, beta = 0.0, gamma = 0.0;
        if (!frozen) {
            tau = sqrt(theta * phi) / rho;                      /* L807 */
            if (phi <= 1e-300) {
                if (!freeze) { outcome = OR_Y_VANISHED; goto done; }
                if (!stopped) { outcome = OR_Y_VANISHED; stopped = 1; }
                frozen = 1;
            } else if (tau - 1.0 <= 1e-14) {
                if (!freeze) { outcome = OR_STAGNATION; goto done; }
                if (!stopped) { outcome = OR_STAGNATION; stopped = 1; }
                frozen = 1;
            } else {
                beta = 1.0 / ((tau - 1.0) * (tau + 1.0));        /* L807-808 */
                gamma = (theta / rho) * beta;                    /* L809 (R1) */
            }
        }
        /* p = beta p + gamma WIy; theta = p^T (WI p); x = x + p  (L811-813) */
        #pragma omp parallel for num_threads(g_threads) schedule(static) if (g_threads > 1)
        for (int64_t j = 0; j < n; ++j) p[j] = beta * p[j] + gamma * wy[j];
        theta = wdot(n, p, wi);
        #pragma omp parallel for num_threads(g_threads) schedule(static) if (g_threads > 1)
        for (int64_t j = 0; j < n; ++j) x[j] = x[j] + p[j];
        if (P_out) for (int64_t j = 0; j < n; ++j) P_out[(size_t)iters * n + j] = p[j];
        iters += 1;
        if (rk) { rk[2] = phi; rk[3] = psi; rk[4] = theta; rk[5] = tau; rk[6] = beta; rk[7] = gamma; }
    }
    if (!stopped) outcome = OR_MAXIT;
done:
    *iters_out = iters;
    free(r); free(y); free(wy); free(p); free(Ap);
    return outcome;
}
