#!/bin/bash
# every bench line of the round-end pass (no tests, no ncu)
set -u
TAG=${1:-b}
mkdir -p gpurun_out
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
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}_c5b.json 2>/dev/null; echo "c5 again rc=$?"
