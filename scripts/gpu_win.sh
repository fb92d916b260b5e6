#!/bin/bash
# Window-kernel check: GPU tests (window first), then a bench sweep of variants.
set -u
mkdir -p gpurun_out
TAG=${1:-win}
timeout 600 python -m pytest tests/test_gpu_window.py -x -q > gpurun_out/pytest_win_${TAG}.log 2>&1; echo "pytest win rc=$?"
tail -15 gpurun_out/pytest_win_${TAG}.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_${TAG}.log
timeout 900 python scripts/sweep.py default,w16,w24,w32s4 --steps 50 --profile-steps 3
timeout 300 python scripts/sweep.py default --steps 50 --profile-steps 3 --no-window
for w in "PLSS_WIN1=2048 PLSS_WIN2=12288" "PLSS_WIN1=8192 PLSS_WIN2=20480"; do
  echo "== $w"; env $w timeout 600 python scripts/sweep.py default --steps 50 --profile-steps 3
done
timeout 600 python scripts/sweep.py default,w16 --steps 50 --profile-steps 3 --workload C3
timeout 600 python scripts/sweep.py default --steps 50 --profile-steps 3 --workload C3 --no-window
