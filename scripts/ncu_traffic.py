"""Per-launch DRAM traffic of K1 / K2 from an `ncu --set full` report -> profiles/*_traffic_*.json
(the `roofline.traffic` figure bench.py reports).  usage: ncu_traffic.py REPORT.ncu-rep SOURCE-NOTE"""
import csv
import json
import re
import subprocess
import sys

KIND = re.compile(r"k_(?:spmv|sellw?)<(\d)|k_rp_(spmm|gen|gram|update)|k_kz_(gemv|resid)")
NAME = {"1": "k1_spmv_csr_resid", "2": "k2_spmv_csc_gather", "3": "k2_spmv_csc_gather",
        "spmm": "rp_spmm_AtS", "gen": "rp_sketch_gen", "gram": "rp_gram", "update": "rp_update",
        "gemv": "kz_gemv_history", "resid": "kz_resid"}


def main(path, note):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    col = {h: i for i, h in enumerate(hdr)}
    acc = {}
    for r in rows[2:]:
        m = KIND.search(r[col["Kernel Name"]])
        key = m and (m.group(1) or m.group(2) or m.group(3))
        if not key or key not in NAME:
            continue
        k = NAME[key]
        rd = float(r[col["dram__bytes_read.sum"]].replace(",", ""))
        wr = float(r[col["dram__bytes_write.sum"]].replace(",", ""))
        t = float(r[col["gpu__time_duration.sum"]].replace(",", ""))
        a = acc.setdefault(k, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += rd
        a[2] += wr
        a[3] += t
    # units: ncu raw reports bytes and ns when --csv without --print-units base? normalise below
    units = rows[1]
    scale_b = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    ub = scale_b.get(units[col["dram__bytes_read.sum"]], 1.0)
    uw = scale_b.get(units[col["dram__bytes_write.sum"]], 1.0)
    ut = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "nsecond": 1e-9, "ms": 1e-3, "msecond": 1e-3}.get(
        units[col["gpu__time_duration.sum"]], 1e-9)
    res = {"source": note, "per_launch": {}}
    for k, (c, rd, wr, t) in acc.items():
        res["per_launch"][k] = {"launches_averaged": c, "dram_bytes": (rd * ub + wr * uw) / c,
                                "dram_read_bytes": rd * ub / c, "dram_write_bytes": wr * uw / c,
                                "duration_s_cold": t * ut / c}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
