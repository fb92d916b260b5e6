"""DRAM traffic per step of each kernel class from an `ncu --set full` report of whole steps ->
profiles/*_traffic_*.json (the `roofline.traffic` figure bench.py reports).

    usage: ncu_traffic.py REPORT.ncu-rep STEPS SOURCE-NOTE

A class's launches may be several kernels per step (K1 of a globally sorted segment = k_sell + its
long rows' k_longchunks; K1 / K2 of S row slabs = S launches each): their bytes are summed over the
report and divided by the number of steps captured."""
import csv
import json
import re
import subprocess
import sys

KIND = re.compile(r"k_(?:spmv|sellw?|longrows|longchunks|scalar)<(\d)|k_(pxupdate)|k_rp_(spmm|gen|gram|update)|k_kz_(gemv|resid)")
NAME = {"1": "k1_spmv_csr_resid", "2": "k2_spmv_csc_gather", "3": "k2_spmv_csc_gather", "pxupdate": "k3_pxupdate",
        "spmm": "rp_spmm_AtS", "gen": "rp_sketch_gen", "gram": "rp_gram", "update": "rp_update",
        "gemv": "kz_gemv_history", "resid": "kz_resid"}
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
TSCALE = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
EXTRA = ["lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__m_xbar2l1tex_read_bytes.sum"]


def main(path, steps, note):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}

    def val(r, name):
        v = float(r[col[name]].replace(",", ""))
        u = units[col[name]]
        return v * (TSCALE.get(u, 1.0) if name.startswith("gpu__time") else SCALE.get(u, 1.0))

    acc = {}
    for r in rows[2:]:
        m = KIND.search(r[col["Kernel Name"]])
        key = m and next(g for g in m.groups() if g)
        if not key or key not in NAME:
            continue
        a = acc.setdefault(NAME[key], {"launches": 0, "kernels": set(), "rd": 0.0, "wr": 0.0, "t": 0.0,
                                       **{e: 0.0 for e in EXTRA if e in col}})
        a["launches"] += 1
        a["kernels"].add(r[col["Kernel Name"]].split("(")[0])
        a["rd"] += val(r, "dram__bytes_read.sum")
        a["wr"] += val(r, "dram__bytes_write.sum")
        a["t"] += val(r, "gpu__time_duration.sum")
        for e in EXTRA:
            if e in col:
                a[e] += float(r[col[e]].replace(",", "")) * SCALE.get(units[col[e]], 1.0)
    res = {"source": note, "steps": steps, "per_step": {}}
    for k, a in acc.items():
        d = {"launches": a["launches"], "kernels": sorted(a["kernels"]), "dram_bytes": (a["rd"] + a["wr"]) / steps,
             "dram_read_bytes": a["rd"] / steps, "dram_write_bytes": a["wr"] / steps,
             "duration_s_cold": a["t"] / steps}
        if "lts__t_sectors_srcunit_tex_op_read.sum" in a:
            d["l2_read_sectors"] = a["lts__t_sectors_srcunit_tex_op_read.sum"] / steps
        if "l1tex__m_xbar2l1tex_read_bytes.sum" in a:
            d["l2_to_sm_bytes"] = a["l1tex__m_xbar2l1tex_read_bytes.sum"] / steps
        res["per_step"][k] = d
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3])
