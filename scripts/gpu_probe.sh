#!/bin/bash
mkdir -p gpurun_out
for cfg in "0 12 -1" "0 12 32" "0 12 64" "6 6 32"; do
  timeout 300 python scripts/rp_spmm_probe.py $cfg 2>&1 | grep -E "granularity|set:|now:|spmm_ms"
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct -k regex:k_rp_spmm -c 1 \
     python scripts/rp_spmm_probe.py $cfg 2>&1 | grep -E "duration|dram__bytes|hit_rate" | head -4
done
