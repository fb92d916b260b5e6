"""paper_2207_07615_b200 -- B200-native hot path of PLSS (arXiv 2207.07615, Algorithm 1).

The product is libplss.so (csrc/, C ABI in include/plss.h): fp64 sm_100a kernels for the
residual-sketch iteration r <- r - A p, y = A^T r, p <- beta p + gamma y, x <- x + p (with an
optional diagonal WI: PLSS W), plus a row-block NCCL path, and randomized projection (eq:pkLong
with a fresh Gaussian sketch, the paper's comparison method) PLSS Kaczmarz (section 7) and the
general growing-sketch engine (section 2.4). `plss` is the thin Python binding (same names as the C ABI).
"""
from .plss import (  # noqa: F401
    Ctx, Matrix, PlssError, load_library, plss_create, plss_create_dist, plss_destroy, plss_finish,
    plss_get_unique_id, plss_profile, plss_query, plss_solve, plss_spmv, plss_spmvT, plss_start, plss_step,
    plss_workspace_bytes, plss_set_wi, plss_column_norms, SYMBOLS, REC, OUTCOMES,
    plss_rp_solve, plss_rp_start, plss_rp_step, plss_rp_finish, plss_rp_sketch, plss_spmmT, plss_rp_profile, rp_ld,
    plss_kz_solve, plss_kz_start, plss_kz_step, plss_kz_finish, plss_kz_profile,
    plss_eg_solve, plss_eg_start, plss_eg_step, plss_eg_finish, plss_eg_profile,
    plss_true_residual, plss_peer_reduce_emulate, plss_create_dist_cols, plss_debug_cta_times, plss_query_segment,
)
