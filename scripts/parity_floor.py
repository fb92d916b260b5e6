#!/usr/bin/env python
"""The fp64 parity floor of the parity configs (DESIGN R11): the oracle against
row-permuted copies of itself (same A and b, rows in another order: another valid summation order of
every dot product and every A^T r column sum), over several permutations. Calls only oracle/ and
plss_gen (input synthesis); writes tests/golden/parity_floor.json, which the GPU parity tests read
to pick the comparison window of each config.

For each config and permutation: K_f = the first k where the two relative-residual histories differ
by more than 1e-11 (100x below the 1e-9 bar), the iteration-count difference, and the final-x
difference ||x_perm - x|| / ||x|| after the config's own cap. For the ill-conditioned configs (C4s,
C4xs) the distribution is wider: 4x the permutations plus the threaded oracle (the same algorithm
with its dot products summed in T fixed blocks, T = 2 .. 32: another valid summation order, the kind
of difference the GPU's tree reductions make), and the x difference as a function of the cap, to
find the window where the 1e-7 x bar has 100x headroom.

    python scripts/parity_floor.py [--perms 5] [--configs C1,C2s,...]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import plss_gen  # noqa: E402

CONFIGS = {"C1": {}, "C2s": {}, "C2": {}, "C4s": {"maxit": 400, "ill": True}, "C4xs": {"ill": True}, "C5xs": {},
           "C5s": {}, "C3_128": {"cfg": ("C3", {"N": 128})}}
CAPS = (10, 15, 20, 25, 30, 40, 50, 75, 100, 150, 200, 300, 400)


def permuted(s, seed):
    perm = np.random.default_rng(seed).permutation(s.m)
    A = s.scipy_csr()[perm]
    A.sort_indices()
    return plss_gen._finish("perm", s.m, s.n, A.indptr, A.indices, A.data, None, s.tol, s.tol_mode,
                            s.maxit, b=s.b[perm], freeze=s.freeze)


def floor_of(name, perms, wi=False):
    spec = CONFIGS[name]
    cfg, kw = spec.get("cfg", (name, {}))
    s = plss_gen.make_config(cfg, **kw)
    if "maxit" in spec:
        s.maxit = spec["maxit"]
    w = oracle.column_norms(s.n, s.col_ptr, s.val_t) if wi else None
    ref = oracle.plss_system(s, wi=w)
    out = {"iters": ref["iters"], "outcome": ref["outcome"], "perms": []}
    nx = np.linalg.norm(ref["x"]) or 1.0
    capped = spec.get("ill", False)
    variants = [("perm", p) for p in range(perms * (4 if capped else 1))]
    if capped:
        variants += [("threads", T) for T in (2, 3, 4, 8, 16, 32)]
    for kind, p in variants:
        if kind == "perm":
            t = permuted(s, 1000 + p)
            other = oracle.plss_system(t, wi=w, maxit=ref["rec"].shape[0] - 1)
        else:
            t = s
            with oracle.threads(p):
                other = oracle.plss_system(t, wi=w, maxit=ref["rec"].shape[0] - 1)
        h0, h1 = ref["hist"], other["hist"]
        k = min(len(h0), len(h1))
        rel = np.abs(h0[:k] - h1[:k]) / np.maximum(h0[:k], 1e-300)
        bad = np.nonzero(rel > 1e-11)[0]
        rec = {"variant": f"{kind} {p}", "iters": int(other["iters"]),
               "kf": int(bad[0]) if bad.size else k, "diters": int(abs(other["iters"] - ref["iters"])),
               "dx": float(np.linalg.norm(other["x"] - ref["x"]) / nx),
               "max_rel_hist_50": float(rel[:50].max()) if k else 0.0}
        if capped:
            rec["dx_at_cap"] = {}
            for cap in CAPS:
                if cap > min(s.maxit, ref["iters"]):
                    break
                a = oracle.plss_system(s, wi=w, maxit=cap)
                with oracle.threads(p if kind == "threads" else 1):
                    b = oracle.plss_system(t, wi=w, maxit=cap)
                rec["dx_at_cap"][cap] = float(np.linalg.norm(b["x"] - a["x"]) / (np.linalg.norm(a["x"]) or 1.0))
        out["perms"].append(rec)
    out["kf_min"] = min(r["kf"] for r in out["perms"])
    out["diters_max"] = max(r["diters"] for r in out["perms"])
    out["dx_max"] = max(r["dx"] for r in out["perms"])
    if capped:
        out["dx_at_cap_max"] = {str(c): max(r["dx_at_cap"][c] for r in out["perms"]) for c in out["perms"][0]["dx_at_cap"]}
        ok = [c for c, v in out["dx_at_cap_max"].items() if v <= 1e-9]
        out["x_window"] = int(max(int(c) for c in ok)) if ok else 0
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--perms", type=int, default=5)
    ap.add_argument("--configs", default="C1,C2s,C4s,C4xs,C5xs,C5s,C3_128")
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "parity_floor.json"))
    args = ap.parse_args()
    res = {}
    if os.path.exists(args.out):
        with open(args.out) as f:
            res = json.load(f)
    res.setdefault("_about", "oracle vs row-permuted oracle (scripts/parity_floor.py; SURVEY 8c-11, DESIGN R11); "
                             "kf: first k with |h - h_perm| / h > 1e-11; dx: final-x difference; "
                             "x_window: the largest cap whose worst x difference is <= 1e-9")
    for name in args.configs.split(","):
        for wi in (False, True):
            t0 = time.time()
            key = name + ("_W" if wi else "")
            res[key] = floor_of(name, args.perms, wi=wi)
            res[key]["perms_n"] = args.perms
            print(f"{key}: kf_min {res[key]['kf_min']} diters_max {res[key]['diters_max']} dx_max {res[key]['dx_max']:.2e}"
                  f" x_window {res[key].get('x_window')} ({time.time() - t0:.0f} s)", flush=True)
            with open(args.out, "w") as f:
                json.dump(res, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
