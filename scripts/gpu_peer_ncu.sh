mkdir -p gpurun_out
CMD="python bench.py --force-dist --dist-step peer --no-cpu-baseline --steps 4 --warmup 3 --profile-steps 1"
$CMD > gpurun_out/peer_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_peer|k_dots|k_pxupdate' -c 60 --csv \
  --log-file gpurun_out/peer_launches.csv $CMD > /dev/null 2>&1; echo "list rc=$?"
ncu --set full --clock-control none -k regex:k_peer_reduce -s 8 -c 2 -o gpurun_out/prof_peer -f $CMD > /dev/null 2>&1; echo "full rc=$?"
