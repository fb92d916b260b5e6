#!/bin/bash
# fail fast: every step under a short timeout; stop at the first timeout
set -u
mkdir -p gpurun_out
run() { timeout "$1" "${@:2}"; rc=$?; if [ $rc -eq 124 ]; then echo "TIMEOUT: ${*:2}"; exit 3; fi; return $rc; }
run 300 python -m pytest tests/test_gpu_window.py -x -q > gpurun_out/pytest_win.log 2>&1; echo "pytest win rc=$?"; tail -3 gpurun_out/pytest_win.log
for e in "X=1" "PLSS_WIN1=0" "PLSS_WIN1=0 PLSS_NSB2=4" "PLSS_WIN1=0 PLSS_NSB2=16" "PLSS_WIN1=0 PLSS_WIN2=12288" "PLSS_WIN1=0 PLSS_WIN2=0"; do
  printf "%-40s " "$e"; env $e timeout 150 python scripts/sweep.py default --steps 30 --profile-steps 3 || exit 3
done
PLSS_WIN1=0 timeout 300 python scripts/sweep.py suw5,wst2 --steps 30 --profile-steps 3
for e in "X=1" "PLSS_WIN1=0 PLSS_WIN2=0"; do
  printf "%-40s " "$e"; env $e timeout 150 python scripts/sweep.py default --steps 30 --profile-steps 3 --workload C3
done
