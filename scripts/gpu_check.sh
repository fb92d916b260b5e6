#!/bin/bash
# One gpurun call: GPU tests, default bench, ncu launch list, ncu --set full of the SpMV kernels.
# usage: scripts/gpu_check.sh TAG [skip-tests]
set -u
TAG=${1:-run}
mkdir -p gpurun_out
if [ "${2:-}" != "skip-tests" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/pytest_${TAG}.log
fi
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_${TAG}.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_(sell|spmv|pxupdate|dots_tail|norm_b|set_nbd)' -c 400 --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --ncu --steps 2 --warmup 1 > gpurun_out/ncu_list_${TAG}.log 2>&1
echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_sell|k_spmv|k_pxupdate' -s 17 -c 5 \
  -o gpurun_out/prof_${TAG} -f python bench.py --ncu --steps 2 --warmup 1 > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu full rc=$?"
