mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kaczmarz.py -q -x > gpurun_out/kz_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/kz_tests.log
for rep in 1 2; do
for lib in libplss_kzold.so libplss.so; do
  PLSS_LIB=$PWD/paper_2207_07615_b200/$lib timeout 600 python bench.py --method kz --no-cpu-baseline > gpurun_out/kz2.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/kz2.json').read().strip().splitlines()[-1]); print('$lib', round(d['value'],1), round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernels_ms_per_step'].items()}, round(d['roofline']['frac'],3))"
done
done
