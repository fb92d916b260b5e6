#!/bin/bash
# A/B of the row-block step on one rank: abd.sh WORKLOAD label [env...]
w=$1; lab=$2; shift 2
env "$@" python bench.py --workload $w --force-dist --steps ${STEPS:-200} --warmup 5 --no-cpu-baseline > gpurun_out/abd_${w}_$lab.json 2> gpurun_out/abd_${w}_$lab.err
python - "$w" "$lab" <<'PY'
import json,sys
w,lab=sys.argv[1:3]
try:
    d=json.loads(open(f"gpurun_out/abd_{w}_{lab}.json").read().strip().splitlines()[-1])
    k=d["kernels_ms_per_step"]
    print(f"{w:6s} {lab:10s} {d['ms_per_step']:.4f} ms/step  " + " ".join(f"{a} {b:.4f}" for a,b in k.items()) + f"  clk {d['clocks']['sm_mhz']}")
except Exception as e:
    print(w, lab, "FAILED", e, open(f"gpurun_out/abd_{w}_{lab}.err").read()[-600:])
PY
