"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: libplss kernels only."""
import csv
import re
import sys
from collections import defaultdict

OURS = re.compile(r"k_(?:spmv|sellw?|longrows|longchunks|scalar)<(\d)[^>]*>|k_rp_[a-z]+|k_kz_[a-z]+|k_eg_[a-zT]+|k_pxupdate|k_norm_b|k_dots_tail|k_set_nbd|k_tile_|k_scan_|k_slab_|k_validate")
ROLE = {"0": "k_spmv<plain>", "1": "k1_spmv_csr_resid", "2": "k2_spmv_csc_gather", "3": "k2_spmv_csc_gather+dots"}


def main(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        m = OURS.search(r["Kernel Name"])
        if not m:
            continue
        name = ROLE[m.group(1)] if m.group(1) else m.group(0)
        rows.append((name, float(r["Metric Value"]), r["Grid Size"], r["Block Size"]))
    agg = defaultdict(lambda: [0, 0.0])
    for name, ns, g, b in rows:
        agg[name][0] += 1
        agg[name][1] += ns
    hot = {k: v for k, v in agg.items() if k.startswith(("k1", "k2", "k_px", "k_dots", "k_rp", "k_kz", "k_eg", "k_spmv<plain>"))}
    tot = sum(v[1] for v in hot.values())
    print(f"{'kernel':32s} {'launches':>8s} {'total us':>10s} {'avg us':>9s} {'share of step':>14s}")
    for k, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        share = f"{100 * ns / tot:.1f}%" if k in hot else "setup"
        print(f"{k:32s} {c:8d} {ns / 1e3:10.1f} {ns / c / 1e3:9.1f} {share:>14s}")


if __name__ == "__main__":
    main(sys.argv[1])
