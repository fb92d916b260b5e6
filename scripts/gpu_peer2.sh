mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_peer.py -q -x > gpurun_out/peer_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/peer_tests.log
for gx in 0 32 74; do
  PLSS_PEER_GX=$gx timeout 600 python bench.py --force-dist --dist-step peer --no-cpu-baseline > gpurun_out/bench_fd_peer_$gx.json 2>/dev/null; echo "gx=$gx rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/bench_fd_peer_$gx.json').read().strip().splitlines()[-1]); print(round(d['value'],2), d['kernels_ms_per_step'])"
done
