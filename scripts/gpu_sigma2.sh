mkdir -p gpurun_out
for rep in 1 2; do
for lib in libplss.so libplss_s1024.so; do
for wl in C4 C5; do
  PLSS_LIB=$PWD/paper_2207_07615_b200/$lib timeout 600 python bench.py --workload $wl --no-cpu-baseline --steps 100 > gpurun_out/sg2.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/sg2.json').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$lib $wl', round(d['ms_per_step'],4), round(k['k1'],4), round(k['k2'],4))" || echo "$lib $wl failed"
done
done
done
