#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python scripts/sweep.py default,pf0,pf1,pf4,w16 --steps 30 --profile-steps 3
timeout 900 python scripts/sweep.py default,pf0,pf4 --steps 30 --profile-steps 3 --no-window
timeout 600 python scripts/sweep.py default,pf0 --steps 30 --profile-steps 3 --workload C3
timeout 600 python scripts/sweep.py default,pf0 --steps 30 --profile-steps 3 --workload C3 --no-window
