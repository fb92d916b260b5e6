"""Probe: Y = A^T S (randomized-projection SpMM, r = 5) on C5-shaped matrices with different
band / uniform mixes, to separate the L2 reuse of the band part from the random uniform part.
usage: python scripts/rp_spmm_probe.py BAND UNIF"""
import sys

import torch

sys.path.insert(0, ".")
import plss_gen  # noqa: E402
import paper_2207_07615_b200 as pkg  # noqa: E402

band, unif = int(sys.argv[1]), int(sys.argv[2])
gran = int(sys.argv[3]) if len(sys.argv) > 3 else -1
pkg.load_library()
import ctypes, glob, os  # noqa: E401,E402
torch.zeros(1, device="cuda")
cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
rt = ctypes.CDLL(cands[0]) if cands else ctypes.CDLL("libcudart.so")
v = ctypes.c_size_t(0)
rt.cudaDeviceGetLimit(ctypes.byref(v), 5)         # cudaLimitMaxL2FetchGranularity
print("default L2 fetch granularity:", v.value, flush=True)
if gran >= 0:
    print("set:", rt.cudaDeviceSetLimit(5, ctypes.c_size_t(gran)), flush=True)
    rt.cudaDeviceGetLimit(ctypes.byref(v), 5)
    print("now:", v.value, flush=True)
d = plss_gen.make_c5_torch(device="cuda", band=band, unif=unif)
A = pkg.Matrix(d["m"], d["n"], d["row_ptr"], d["col_idx"], d["val"], d["col_ptr"], d["row_idx"], d["val_t"])
ctx = pkg.plss_create(A, slabs=1, sell=False, maxit_cap=4)
S = pkg.plss_rp_sketch(ctx, 5, seed=3, k=1)
Y = pkg.plss_spmmT(ctx, S, r=5)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    pkg.plss_spmmT(ctx, S, r=5, Y=Y)
e1.record()
torch.cuda.synchronize()
print(f"band={band} unif={unif} gran={gran} nnz={A.nnz} spmm_ms={e0.elapsed_time(e1) / 3:.3f}", flush=True)
