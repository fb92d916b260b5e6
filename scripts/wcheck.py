"""Debug: the failing window case (C5xs, slabs=3, spmvT) with the WCHECK build."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PLSS_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2207_07615_b200", "libplss_wcheck.so")
import numpy as np, torch, plss_gen, oracle
import paper_2207_07615_b200 as pkg
pkg.load_library()
s = plss_gen.make_config("C5xs")
A = pkg.Matrix.from_arrays(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t)
ctx = pkg.plss_create(A, slabs=3, maxit_cap=4, validate=True)
print(pkg.plss_query(ctx), flush=True)
u = np.random.default_rng(3).standard_normal(s.m)
v = torch.empty(s.n, dtype=torch.float64, device="cuda")
pkg.plss_spmvT(ctx, torch.from_numpy(u).cuda(), v)
torch.cuda.synchronize()
ref = oracle.spmvT(s.n, s.col_ptr, s.row_idx, s.val_t, u)
bad = np.nonzero(v.cpu().numpy() != ref)[0]
print("bad", bad[:20], len(bad), flush=True)
