mkdir -p gpurun_out
CMD="python bench.py --ncu --steps 2 --warmup 1"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_sell<|k_spmv<|k_pxupdate' -s 8 -c 6 \
  -o gpurun_out/prof_c5s10 -f $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
