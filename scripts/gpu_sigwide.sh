mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_window.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py tests/test_gpu_engine.py tests/test_gpu_peer.py -q -x > gpurun_out/sw_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/sw_tests.log
for rep in 1 2; do
for sw in 1 0; do
for wl in C4 C4alt C5; do
  PLSS_SIGWIDE=$sw timeout 600 python bench.py --workload $wl --no-cpu-baseline --steps 100 > gpurun_out/sw.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('sigwide=$sw $wl', round(d['ms_per_step'],4), round(k['k1'],4), round(k['k2'],4))"
done
done
done
