#!/bin/bash
set -u
for e in "PLSS_WIN1=0 PLSS_WIN2=0" "PLSS_WIN1=0 PLSS_L1WIN=2" "PLSS_WIN1=0 PLSS_WIN2=32768 PLSS_L1WIN=2" \
         "PLSS_WIN1=0 PLSS_WIN2=8192 PLSS_L1WIN=2" "PLSS_L1WIN=3" "PLSS_WIN2=0 PLSS_L1WIN=1" "PLSS_WIN1=0 PLSS_WIN2=0 PLSS_SELLC=1"; do
  printf "%-50s " "$e"; env $e timeout 300 python scripts/sweep.py default --steps 30 --profile-steps 3
done
for e in "PLSS_WIN1=0 PLSS_WIN2=0" "PLSS_L1WIN=3"; do
  printf "%-50s " "$e"; env $e timeout 300 python scripts/sweep.py default --steps 30 --profile-steps 3 --workload C3
done
