mkdir -p gpurun_out
for rep in 1 2; do
for lib in libplss.so libplss_s256.so; do
  PLSS_LIB=$PWD/paper_2207_07615_b200/$lib timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/sg.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/sg.json').read().strip().splitlines()[-1]); print('$lib', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"
done
done
