mkdir -p gpurun_out

for rep in 1 2; do
for f in triangular qr; do
  timeout 600 python bench.py --method eg --eg-factor $f --no-cpu-baseline > gpurun_out/eg2_$f.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/eg2_$f.json').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernels_ms_per_step'].items()}, round(d['roofline']['frac'],3))"
done
done
