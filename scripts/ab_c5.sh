#!/bin/bash
# A/B runs of the C5 bench: label, env...
run() { lab=$1; shift; env "$@" python bench.py --steps 30 --warmup 3 --no-cpu-baseline $BARGS > gpurun_out/ab_$lab.json 2> gpurun_out/ab_$lab.err; python - "$lab" <<'PY'
import json,sys
lab=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/ab_{lab}.json").read().strip().splitlines()[-1])
    k=d["kernels_ms_per_step"]
    print(f"{lab:28s} {d['ms_per_step']:.3f} ms/step  frac {d['achieved_frac_of_peak']:.3f}  K1 {k['k1']:.3f} K2 {k['k2']:.3f} K3 {k['k3']:.3f}  clk {d['clocks']['sm_mhz']}")
except Exception as e:
    print(lab, "FAILED", e, open(f"gpurun_out/ab_{lab}.err").read()[-500:])
PY
}
OLD=$PWD/paper_2207_07615_b200/libplss_old.so
run old PLSS_LIB=$OLD
run new_l0_s0 PLSS_LOCW=0 PLSS_STAT=0
run new_l16k_s0 PLSS_LOCW=16384 PLSS_STAT=0
run new_l0_s1 PLSS_LOCW=0 PLSS_STAT=1
L=$PWD/paper_2207_07615_b200
run def
run yq6 PLSS_LIB=$L/libplss_yq6.so
run yq4 PLSS_LIB=$L/libplss_yq4.so
run def2
run yq6b PLSS_LIB=$L/libplss_yq6.so
