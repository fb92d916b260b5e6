mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_fullsize.py -q -x -k "engine or eg" > gpurun_out/eg_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/eg_tests.log
for rep in 1 2; do
for f in triangular qr; do
  timeout 600 python bench.py --method eg --eg-factor $f --no-cpu-baseline > gpurun_out/eg3_$f.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/eg3_$f.json').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernels_ms_per_step'].items()}, round(d['roofline']['frac'],3))"
done
done
