#!/bin/bash
# A/B of library variants: interleaved repeats (run-to-run spread is 5-10%), C5 unless $WL set
set -u
VARS=$1; REP=${2:-3}; WL=${WL:-C5}
for r in $(seq $REP); do
  timeout 600 python scripts/sweep.py $VARS --steps 60 --profile-steps 3 --workload $WL
done
