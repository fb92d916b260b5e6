#!/bin/bash
set -u
export PLSS_WIN1=0 PLSS_WIN2=0
timeout 300 python scripts/sweep.py default,abl4 --steps 30 --profile-steps 3
timeout 300 python scripts/sweep.py default,abl4 --steps 30 --profile-steps 3 --slabs 1
PLSS_WIN1=4096 PLSS_WIN2=16384 timeout 300 python scripts/sweep.py wst8 --steps 30 --profile-steps 3
