#!/bin/bash
set -u
export PLSS_WIN1=0 PLSS_WIN2=0
for sl in 8 16; do
  timeout 600 python scripts/sweep.py default,h2,noh --steps 30 --profile-steps 3 --slabs $sl
done
PLSS_SELLC=1 timeout 600 python scripts/sweep.py default,h2 --steps 30 --profile-steps 3
timeout 600 python scripts/sweep.py default,h2,noh --steps 30 --profile-steps 3 --slabs 12
timeout 600 python scripts/sweep.py default,noh --steps 30 --profile-steps 3 --workload C3
