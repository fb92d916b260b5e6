#!/bin/bash
# Round-end refresh: full GPU suite, smoke, every bench line, ncu launch lists and full captures.
set -u
TAG=${1:-fin}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_${TAG}.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
timeout 600 python bench.py --method rp > gpurun_out/bench_${TAG}_rp.json 2>/dev/null; echo "rp rc=$?"
timeout 600 python bench.py --method kz > gpurun_out/bench_${TAG}_kz.json 2>/dev/null; echo "kz rc=$?"
timeout 600 python bench.py --method eg > gpurun_out/bench_${TAG}_eg.json 2>/dev/null; echo "eg rc=$?"
timeout 600 python bench.py --method eg --eg-factor qr --no-cpu-baseline > gpurun_out/bench_${TAG}_egqr.json 2>/dev/null; echo "egqr rc=$?"
for v in "ar:--dist-step allreduce" "peer:--dist-step peer" "rsag:--dist-step rsag"; do
  timeout 600 python bench.py --force-dist --no-cpu-baseline ${v#*:} > gpurun_out/bench_${TAG}_fd_${v%%:*}.json 2>/dev/null; echo "fd ${v%%:*} rc=$?"
done
timeout 600 python bench.py --workload C4 --force-dist --partition cols --no-cpu-baseline > gpurun_out/bench_${TAG}_c4_cols.json 2>/dev/null; echo "c4 cols rc=$?"
timeout 600 python bench.py --workload C4 --no-cpu-baseline > gpurun_out/bench_${TAG}_c4.json 2>/dev/null; echo "c4 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_ref.json 2>/dev/null; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_(sell|spmv|pxupdate|dots_tail|norm_b|set_nbd)' -c 400 --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --ncu --steps 2 --warmup 1 > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_sell<|k_spmv<|k_pxupdate' -s 8 -c 6 \
  -o gpurun_out/prof_${TAG} -f python bench.py --ncu --steps 2 --warmup 1 > /dev/null 2>&1; echo "ncu full rc=$?"
