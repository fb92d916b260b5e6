mkdir -p gpurun_out
for v in "single:" "rows:--force-dist" "cols:--force-dist --partition cols"; do
  name=${v%%:*}; flags=${v#*:}
  timeout 900 python bench.py --workload C4 --no-cpu-baseline $flags > gpurun_out/bench_c4_$name.json 2> gpurun_out/bench_c4_$name.err; echo "$name rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/bench_c4_$name.json').read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],4), d['config']['parallelism'], d['kernels_ms_per_step'], d['gpu_launches'])" || tail -5 gpurun_out/bench_c4_$name.err
done
