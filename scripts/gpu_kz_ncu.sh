mkdir -p gpurun_out
CMD="python bench.py --method kz --ncu --steps 200 --warmup 3"
$CMD > gpurun_out/kzn_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_kz_resid' -s 150 -c 2 \
  -o gpurun_out/prof_kzres -f $CMD > gpurun_out/kzn.log 2>&1; echo "ncu rc=$?"
