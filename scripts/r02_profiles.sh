#!/bin/bash
# Round-2 evidence on one B200: bench lines (C5 default run + reference arm, C4, C3), the launch
# list of the C5 bench command, and one `ncu --set full` capture of a whole step for C5, C4, C3
# (each command runs once without ncu first). Outputs under gpurun_out/r02_*.
set -u
K='regex:k_sell|k_pxupdate|k_longrows|k_longchunks|k_scalar'
python bench.py > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_bench_c5.err
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r02_bench_c5_reference.json 2>/dev/null
for w in C4 C3 C4alt; do
  python bench.py --workload $w > gpurun_out/r02_bench_${w,,}.json 2> gpurun_out/r02_bench_${w,,}.err
done
python bench.py --ncu --steps 2 --warmup 1 > gpurun_out/r02_ncu_plain_c5.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c5.csv \
      python bench.py --ncu --steps 2 --warmup 1 > /dev/null 2>&1
python bench.py --ncu --steps 2 --warmup 1 > gpurun_out/r02_ncu_plain_c5b.log 2>&1 && \
  ncu --set full --import-source on --clock-control none -k "$K" -s 21 -c 21 -o gpurun_out/r02_full_c5 \
      python bench.py --ncu --steps 2 --warmup 1 > gpurun_out/r02_ncu_c5.log 2>&1
for w in C4 C3; do
  n=4; [ $w = C3 ] && n=3
  python bench.py --workload $w --ncu --steps 2 --warmup 1 > gpurun_out/r02_ncu_plain_$w.log 2>&1 && \
    ncu --set full --import-source on --clock-control none -k "$K" -s $n -c $n -o gpurun_out/r02_full_${w,,} \
        python bench.py --workload $w --ncu --steps 2 --warmup 1 > gpurun_out/r02_ncu_$w.log 2>&1
done
ls -la gpurun_out/r02_full_* gpurun_out/r02_launches_c5.csv
