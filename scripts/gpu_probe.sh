#!/bin/bash
# RP A^T S DRAM bytes per random S-row gather for L2 prefetch-size variants (PLSS_LIB selects the build)
mkdir -p gpurun_out
for lib in libplss.so; do
  export PLSS_LIB=$PWD/paper_2207_07615_b200/$lib
  echo "== $lib"
  timeout 300 python scripts/rp_spmm_probe.py 0 12 2>&1 | grep spmm_ms
  timeout 300 python scripts/rp_spmm_probe.py 6 6 2>&1 | grep spmm_ms
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum -k regex:k_rp_spmm -c 1 \
     python scripts/rp_spmm_probe.py 0 12 2>&1 | grep -E "duration|dram__bytes" | head -2
done
