mkdir -p gpurun_out
for rep in 1 2 3; do
for ov in 0 1; do
  PLSS_OVERLAP=$ov timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/ov.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ov.json').read().strip().splitlines()[-1]); print('ov=$ov', round(d['ms_per_step'],4), round(d['final_hist'],20), d['clocks']['sm_mhz'])"
done
done
