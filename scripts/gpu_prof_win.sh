#!/bin/bash
# ncu --set full of the windowed kernels (C5: K1 slab 0, K2 slab 0) and a short sweep.
set -u
mkdir -p gpurun_out
TAG=${1:-pw}
timeout 600 python scripts/sweep.py default,w16 --steps 30 --profile-steps 3
timeout 600 python scripts/sweep.py default --steps 30 --profile-steps 3 --workload C3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_sellw' -s 16 -c 4 \
  -o gpurun_out/prof_${TAG} -f python bench.py --ncu --steps 2 --warmup 1 > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_sellw' -s 4 -c 2 \
  -o gpurun_out/prof_${TAG}_c3 -f python bench.py --ncu --steps 2 --warmup 1 --workload C3 > gpurun_out/ncu_full_${TAG}_c3.log 2>&1
echo "ncu c3 rc=$?"
