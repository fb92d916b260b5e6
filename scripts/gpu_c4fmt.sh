mkdir -p gpurun_out
for rep in 1 2; do
for wl in C4 C4alt; do
for sc in 2 1 0; do
  PLSS_SELLC=$sc timeout 600 python bench.py --workload $wl --no-cpu-baseline --steps 200 > gpurun_out/c4f.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/c4f.json').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$wl sellc=$sc', round(d['ms_per_step'],4), 'k1', round(k['k1'],4), 'k2', round(k['k2'],4))"
done
done
done
