mkdir -p gpurun_out
CMD="python bench.py --workload C4 --ncu --steps 3 --warmup 1"
$CMD > gpurun_out/c4n_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k regex:'k_sell<' -s 2 -c 2 \
  -o gpurun_out/prof_c4 -f $CMD > gpurun_out/c4n.log 2>&1; echo "ncu rc=$?"
