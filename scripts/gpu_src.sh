#!/bin/bash
set -u
mkdir -p gpurun_out
export PLSS_WIN1=0
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_sellw' -s 8 -c 1 \
  -o gpurun_out/prof_src_w -f python bench.py --ncu --steps 2 --warmup 1 > gpurun_out/ncu_src_w.log 2>&1
echo "ncu rc=$?"
export PLSS_WIN2=0
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_sell' -s 17 -c 2 \
  -o gpurun_out/prof_src_p -f python bench.py --ncu --steps 2 --warmup 1 > gpurun_out/ncu_src_p.log 2>&1
echo "ncu rc=$?"
