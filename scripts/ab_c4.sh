#!/bin/bash
# A/B runs of the C4 bench: label, env...
run() { lab=$1; shift; env "$@" python bench.py --workload C4 --steps 200 --warmup 5 --no-cpu-baseline $BARGS > gpurun_out/ab4_$lab.json 2> gpurun_out/ab4_$lab.err; python - "$lab" <<'PY'
import json,sys
lab=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/ab4_{lab}.json").read().strip().splitlines()[-1])
    k=d["kernels_ms_per_step"]
    print(f"{lab:28s} {d['ms_per_step']:.4f} ms/step  frac {d['achieved_frac_of_peak']:.3f}  K1 {k['k1']:.4f} K2 {k['k2']:.4f} K3 {k['k3']:.4f}  clk {d['clocks']['sm_mhz']}")
except Exception as e:
    print(lab, "FAILED", e, open(f"gpurun_out/ab4_{lab}.err").read()[-500:])
PY
}

run def
BARGS="--workload C4alt"
run alt_def
BARGS=""
run def2
