mkdir -p gpurun_out
for rep in 1 2; do
for lib in libplss.so libplss_rt4k.so; do
  PLSS_LIB=$PWD/paper_2207_07615_b200/$lib timeout 600 python bench.py --method eg --no-cpu-baseline > gpurun_out/egrt.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/egrt.json').read().strip().splitlines()[-1]); print('$lib', round(d['value'],1), round(d['kernels_ms_per_step']['gemvT'],4))"
done
done
