#!/bin/bash
# Round-2 final evidence on one B200, from the final build: the GPU suite and smoke(), one
# `ncu --set full` capture of a whole loop step for C5, C4, C3 (each command run once without ncu
# first) summarised on the box (reports are deleted: gpurun_out/ must stay under 64 MiB), the
# per-step traffic JSON bench.py reads for roofline.traffic, the launch list of the C5 bench command,
# then the bench lines (C5 default run + reference arm, C4, C3, C4-alt). Outputs: gpurun_out/r02_*.
set -u
K='regex:k_sell|k_pxupdate|k_longrows|k_longchunks|k_scalar'
python -m pytest tests -m gpu -q > gpurun_out/r02_pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.txt 2>&1
for w in C5 C4 C3; do
  case $w in C5) n=21 ;; C4) n=4 ;; C3) n=3 ;; esac
  lw=${w,,}
  python bench.py --workload $w --ncu --steps 2 --warmup 1 > gpurun_out/r02_ncu_plain_$lw.log 2>&1 && \
    ncu --set full --import-source on --clock-control none -k "$K" -s $n -c $n -o /tmp/r02_full_$lw \
        python bench.py --workload $w --ncu --steps 2 --warmup 1 > gpurun_out/r02_ncu_$lw.log 2>&1
  python scripts/ncu_summary.py /tmp/r02_full_$lw.ncu-rep > gpurun_out/r02_ncu_full_$lw.txt
  python scripts/ncu_hot_sass.py /tmp/r02_full_$lw.ncu-rep > gpurun_out/r02_ncu_hot_sass_$lw.txt 2>&1
  python scripts/ncu_traffic.py /tmp/r02_full_$lw.ncu-rep 1 "gpurun $(date -u +%F), ncu --set full --clock-control none -k $K -s $n -c $n (one whole loop step), bench.py --workload $w --ncu --steps 2 --warmup 1, round-2 final build (scripts/r02_final.sh, scripts/ncu_traffic.py)" \
    > gpurun_out/r02_ncu_traffic_$lw.json && cp gpurun_out/r02_ncu_traffic_$lw.json profiles/
  rm -f /tmp/r02_full_$lw.ncu-rep
done
python bench.py --ncu --steps 2 --warmup 1 > gpurun_out/r02_ncu_plain_launches.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/r02_launches_c5.csv \
      python bench.py --ncu --steps 2 --warmup 1 > /dev/null 2>&1
python scripts/launch_summary.py /tmp/r02_launches_c5.csv > gpurun_out/r02_launches_c5.txt 2>&1
python bench.py > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_bench_c5.err
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r02_bench_c5_reference.json 2>/dev/null
for w in C4 C3 C4alt; do
  python bench.py --workload $w > gpurun_out/r02_bench_${w,,}.json 2> gpurun_out/r02_bench_${w,,}.err
done
du -sh gpurun_out
