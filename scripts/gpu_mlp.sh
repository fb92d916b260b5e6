#!/bin/bash
set -u
export PLSS_WIN1=0 PLSS_WIN2=0
timeout 900 python scripts/sweep.py default,su4m6,su4m8,su6m5,su12m3,su16m2 --steps 30 --profile-steps 3
timeout 600 python scripts/sweep.py default,su4m8,su16m2 --steps 30 --profile-steps 3 --workload C3
