#!/usr/bin/env python
"""Per-CTA balance of the fmt 3 SpMV launches (diagnostics build libplss_dbg.so, -DPLSS_DBGCTA, with
PLSS_DBG_CTA=1): for K1 and K2 of a workload, each persistent CTA's duration, stored entries and
units, sorted by duration; shows which work the straggler CTAs hold.

    PLSS_LIB=paper_2207_07615_b200/libplss_dbg.so PLSS_DBG_CTA=1 python scripts/cta_balance.py --workload C4
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--slab", type=int, default=0)
    ap.add_argument("--all-slabs", action="store_true", help="one line per slab: K1 / K2 max and median CTA us")
    args = ap.parse_args()
    import torch
    import paper_2207_07615_b200 as pkg
    pkg.load_library()
    w = bench.load_workload(args.workload, 0, 1, torch.device("cuda"))
    A = pkg.Matrix(w["m"], w["n"], w["row_ptr"], w["col_idx"], w["val"], w["col_ptr"], w["row_idx"], w["val_t"])
    ctx = pkg.plss_create(A, maxit_cap=16)
    pkg.plss_solve(ctx, w["b"], tol=0.0, maxit=6, flags=1)
    if args.all_slabs:
        S = pkg.plss_query(ctx)["slabs"]
        ev = []
        for sl in range(S):
            for which in (1, 2):
                t = pkg.plss_debug_cta_times(ctx, which, sl)
                ev.append((f"K{which}_{sl}", t[:, 0].min(), t[:, 1].max()))
        t0 = ev[0][1]
        print("timeline of the last step (us from K1_0's first CTA): launch [start, end] gap-before")
        prev = None
        for name, a, b in ev:
            gap = (a - prev) / 1e3 if prev is not None else 0.0
            print(f"   {name:6s} [{(a - t0) / 1e3:8.1f}, {(b - t0) / 1e3:8.1f}]  gap {gap:6.1f}")
            prev = b
        for sl in range(S):
            line = []
            for which in (1, 2):
                t = pkg.plss_debug_cta_times(ctx, which, sl)
                dur = (t[:, 1] - t[:, 0]) / 1e3
                span = (t[:, 1].max() - t[:, 0].min()) / 1e3
                line.append(f"K{which} max {dur.max():6.1f} med {np.median(dur):6.1f} span {span:6.1f}")
            print(f"slab {sl}: " + " | ".join(line))
        pkg.plss_destroy(ctx)
        return
    for which, name in ((1, "K1"), (2, "K2")):
        t = pkg.plss_debug_cta_times(ctx, which, args.slab)
        dur = (t[:, 1] - t[:, 0]) / 1e3
        start = (t[:, 0] - t[:, 0].min()) / 1e3
        order = np.argsort(-dur)
        print(f"{name}: grid {len(t)}  duration us: max {dur.max():.1f} median {np.median(dur):.1f} min {dur.min():.1f}; "
              f"entries total {t[:, 2].sum()} (per CTA median {np.median(t[:, 2]):.0f}); units {t[:, 3].sum()}")
        print("   slowest CTAs: (cta, start us, dur us, entries, units, entries/unit)")
        for c in list(order[:8]) + list(order[-3:]):
            print(f"   {c:4d} {start[c]:7.1f} {dur[c]:7.1f} {t[c, 2]:9d} {t[c, 3]:7d} {t[c, 2] / max(t[c, 3], 1):8.1f}")
        # duration vs position in the unit order (CTA index = unit order)
        q = np.array_split(np.arange(len(t)), 8)
        print("   by CTA octile (unit order): " + "  ".join(f"{dur[i].mean():.0f}us/{t[i, 2].sum() / 1e6:.2f}M/{t[i, 3].sum()}u" for i in q))
    pkg.plss_destroy(ctx)


if __name__ == "__main__":
    main()
