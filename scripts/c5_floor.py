#!/usr/bin/env python
"""The fp64 parity floor of the full-size C5 (the timed config): the oracle on C5 against the
oracle on a row-permuted C5 ("measure K_f on full C5 against a
row-permuted oracle"). Runs on a GPU box: the C5 arrays come from plss_gen.make_c5_torch (the
bench's own generator, input synthesis) and the permutation is index work in torch; every number
written comes from oracle/ (the threaded oracle, oracle_set_threads, on all host cores).

Writes tests/golden/c5_floor.json: per k the relative history difference, K_f (first k > 1e-11),
the final-x difference after `--steps`, and the iterations to each tolerance of both runs.

    python scripts/c5_floor.py [--steps 60] [--seed 1000]
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

TOLS = (1e-4, 1e-6, 1e-8, 1e-10, 1e-12)


def host(d):
    return {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in d.items()}


def permute_rows(d, seed):
    """Rows of C5 in a random order: CSR rows gathered, CSC row indices relabelled and each column
    re-sorted ascending (so the oracle's column sums run in another order); b permuted."""
    import torch
    m, n = d["m"], d["n"]
    per = int(d["row_ptr"][1] - d["row_ptr"][0])
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    perm = torch.randperm(m, generator=g, device="cuda")
    inv = torch.empty_like(perm)
    inv[perm] = torch.arange(m, device="cuda")
    col_idx = d["col_idx"].view(m, per)[perm].reshape(-1)
    val = d["val"].view(m, per)[perm].reshape(-1)
    b = d["b"][perm]
    cnt = (d["col_ptr"][1:] - d["col_ptr"][:-1]).long()
    col_of = torch.repeat_interleave(torch.arange(n, device="cuda"), cnt)
    new_row = inv[d["row_idx"].long()]
    order = torch.sort(col_of * m + new_row, stable=True).indices
    del col_of
    row_idx = new_row[order].to(torch.int32)
    val_t = d["val_t"][order]
    del order, new_row
    return {"m": m, "n": n, "row_ptr": d["row_ptr"], "col_idx": col_idx, "val": val,
            "col_ptr": d["col_ptr"], "row_idx": row_idx, "val_t": val_t, "b": b}


def run_oracle(h, steps):
    t0 = time.time()
    r = oracle.plss(h["m"], h["n"], h["row_ptr"], h["col_idx"], h["val"], h["col_ptr"], h["row_idx"], h["val_t"],
                    h["b"], tol=0.0, maxit=steps, freeze=True)
    return r, time.time() - t0


def iters_to(hist, tol):
    k = np.nonzero(hist <= tol)[0]
    return int(k[0]) if k.size else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--seed", type=int, default=1000)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "c5_floor.json"))
    args = ap.parse_args()
    import torch
    d = plss_gen.make_c5_torch(device="cuda")
    hp = host(permute_rows(d, args.seed))
    torch.cuda.synchronize()
    h = host(d)
    del d
    torch.cuda.empty_cache()
    T = os.cpu_count() or 1
    with oracle.threads(T):
        a, ta = run_oracle(h, args.steps)
        b, tb = run_oracle(hp, args.steps)
    ha, hb = a["rec"][:args.steps, 0], b["rec"][:args.steps, 0]
    rel = np.abs(ha - hb) / np.maximum(ha, 1e-300)
    bad = np.nonzero(rel > 1e-11)[0]
    out = {"about": "full C5 (plss_gen.make_c5_torch, seed 0): threaded oracle vs the same on a row-permuted C5 "
                    "(scripts/c5_floor.py); freeze mode, tol 0",
           "steps": args.steps, "perm_seed": args.seed, "threads": T, "oracle_s": [ta, tb],
           "kf": int(bad[0]) if bad.size else args.steps,
           "rel_hist": rel.tolist(), "hist": ha.tolist(),
           "dx": float(np.linalg.norm(a["x"] - b["x"]) / np.linalg.norm(a["x"])),
           "iters_to": {str(t): [iters_to(ha, t), iters_to(hb, t)] for t in TOLS}}
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k not in ("rel_hist", "hist")}))


if __name__ == "__main__":
    main()
