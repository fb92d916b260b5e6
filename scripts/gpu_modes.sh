#!/bin/bash
# Sweep of SpMV formats per kernel (env overrides read at plss_create).
set -u
mkdir -p gpurun_out
WL=${1:-C5}
for e in "X=1" "PLSS_WIN1=0 PLSS_WIN2=0" "PLSS_WIN1=0 PLSS_WIN2=0 PLSS_SELLC=1" "PLSS_WIN1=0 PLSS_WIN2=0 PLSS_SELLC=2" \
         "PLSS_WIN1=0" "PLSS_WIN1=0 PLSS_WIN2=8192" "PLSS_WIN1=0 PLSS_SELLC=2"; do
  printf "%-45s " "$e"; env $e timeout 300 python scripts/sweep.py default --steps 30 --profile-steps 3 --workload $WL
done
