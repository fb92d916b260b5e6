mkdir -p gpurun_out
for rep in 1 2 3; do
for S in 9 10 11 8; do
  timeout 600 python bench.py --no-cpu-baseline --steps 100 --slabs $S > gpurun_out/sl_$S.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/sl_$S.json').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('S=$S', round(d['ms_per_step'],4), 'k1', round(k['k1'],3), 'k2', round(k['k2'],3), d['clocks']['sm_mhz'])"
done
done
