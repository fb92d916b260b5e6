#!/bin/bash
# Growing-sketch engine (NEXT-4): bench (gaussian sketch), ncu launch list, ncu --set full.
set -u
TAG=${1:-eg}
mkdir -p gpurun_out
timeout 600 python bench.py --method eg > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench_${TAG}.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_eg|k_sell|k_spmv|k_norm_b' -c 600 --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --method eg --ncu --steps 60 --warmup 3 > gpurun_out/ncu_list_${TAG}.log 2>&1
echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_eg_(gemvT|gemv|trit)' -s 150 -c 3 \
  -o gpurun_out/prof_${TAG} -f python bench.py --method eg --ncu --steps 100 --warmup 3 > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu full rc=$?"
