mkdir -p gpurun_out
for rep in 1 2; do
for lib in libplss.so libplss_p2.so libplss_p4.so; do
for wl in C4 C4alt C5; do
  PLSS_LIB=$PWD/paper_2207_07615_b200/$lib timeout 600 python bench.py --workload $wl --no-cpu-baseline --steps 100 > gpurun_out/pair.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/pair.json').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$lib $wl', round(d['ms_per_step'],4), {a: round(b,4) for a,b in k.items()})"
done
done
done
