mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_peer.py tests/test_gpu_dist.py -q -x > gpurun_out/peer_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/peer_tests.log
for step in allreduce peer rsag; do
  timeout 600 python bench.py --force-dist --dist-step $step --no-cpu-baseline > gpurun_out/bench_fd_$step.json 2> gpurun_out/bench_fd_$step.err; echo "bench $step rc=$?"
  tail -c 600 gpurun_out/bench_fd_$step.json | head -c 600; echo
done
