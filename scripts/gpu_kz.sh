#!/bin/bash
# PLSS Kaczmarz (NEXT-3): GPU tests, bench, ncu launch list, ncu --set full of its kernels.
set -u
TAG=${1:-kz}
mkdir -p gpurun_out
if [ "${2:-}" != "skip-tests" ]; then
  timeout 900 python -m pytest tests/test_gpu_kaczmarz.py -x -q > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"
  tail -2 gpurun_out/pytest_${TAG}.log
fi
timeout 600 python bench.py --method kz > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
tail -c 2500 gpurun_out/bench_${TAG}.json; tail -3 gpurun_out/bench_${TAG}.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_kz|k_sell|k_spmv|k_norm_b' -c 400 --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --method kz --ncu --steps 80 --warmup 3 > gpurun_out/ncu_list_${TAG}.log 2>&1
echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_kz_(gemv|resid)' -s 150 -c 4 \
  -o gpurun_out/prof_${TAG} -f python bench.py --method kz --ncu --steps 100 --warmup 3 > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu full rc=$?"
