mkdir -p gpurun_out
for rep in 1 2 3; do
for lib in libplss.so libplss_pel.so; do
  PLSS_LIB=$PWD/paper_2207_07615_b200/$lib timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/pel.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/pel.json').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$lib', round(d['ms_per_step'],4), {a: round(b,4) for a,b in k.items() if b}, d['clocks']['sm_mhz'])"
done
done
