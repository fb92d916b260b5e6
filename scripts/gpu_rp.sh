#!/bin/bash
# Randomized projection (NEXT-2): GPU tests, bench, ncu launch list, ncu --set full of its kernels.
# usage: scripts/gpu_rp.sh TAG [skip-tests]
set -u
TAG=${1:-rp}
mkdir -p gpurun_out
if [ "${2:-}" != "skip-tests" ]; then
  timeout 900 python -m pytest tests/test_gpu_randproj.py "tests/test_gpu_fullsize.py::test_c5_full_randproj_sampled_and_projection" -x -q > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/pytest_${TAG}.log
fi
timeout 600 python bench.py --method rp --steps 20 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
tail -c 2500 gpurun_out/bench_${TAG}.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_rp|k_sell|k_spmv|k_norm_b' -c 200 --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --method rp --ncu --steps 3 --warmup 1 > gpurun_out/ncu_list_${TAG}.log 2>&1
echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_rp_(spmm|gen|gram|update)' -s 8 -c 4 \
  -o gpurun_out/prof_${TAG} -f python bench.py --method rp --ncu --steps 3 --warmup 1 > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu full rc=$?"
