mkdir -p gpurun_out
for rep in 1 2; do
for v in "def:" "ucs128:PLSS_UC_SIG=128" "ucs512:PLSS_UC_SIG=512" "uc64:PLSS_UC=64" "uc256:PLSS_UC=256"; do
  env ${v#*:} timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/uc.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/uc.json').read().strip().splitlines()[-1]); print('${v%%:*}', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"
done
done
