mkdir -p gpurun_out
for rep in 1 2; do
for h in 0 1 3 5 2; do
  PLSS_RHINT=$h timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/rh_$h.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/rh_$h.json').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('rhint=$h', round(d['ms_per_step'],4), 'k1', round(k['k1'],3), 'k2', round(k['k2'],3), d['clocks']['sm_mhz'])"
done
done
