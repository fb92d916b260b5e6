#!/bin/bash
# A/B runs of bench.py: ab.sh WORKLOAD label [env...]; prints one summary line per run.
# Used as: gpurun -- 'bash scripts/ab.sh C4 def; bash scripts/ab.sh C4 v2 PLSS_LIB=...'
w=$1; lab=$2; shift 2
env "$@" python bench.py --workload $w --steps ${STEPS:-200} --warmup 5 --no-cpu-baseline > gpurun_out/ab_${w}_$lab.json 2> gpurun_out/ab_${w}_$lab.err
python - "$w" "$lab" <<'PY'
import json,sys
w,lab=sys.argv[1:3]
try:
    d=json.loads(open(f"gpurun_out/ab_{w}_{lab}.json").read().strip().splitlines()[-1])
    k=d["kernels_ms_per_step"]
    print(f"{w:6s} {lab:20s} {d['ms_per_step']:.4f} ms/step  frac {d['achieved_frac_of_peak']:.3f}  K1 {k['k1']:.4f} K2 {k['k2']:.4f} K3 {k['k3']:.4f}  clk {d['clocks']['sm_mhz']}")
except Exception as e:
    print(w, lab, "FAILED", e, open(f"gpurun_out/ab_{w}_{lab}.err").read()[-800:])
PY
