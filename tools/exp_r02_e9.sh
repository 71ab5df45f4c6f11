set -u
for i in 1 2; do
for v in default SB_LANES=1 SB_LANES=2; do
  if [ $v = default ]; then timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/e9.json 2>/dev/null
  else env $v timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/e9.json 2>/dev/null; fi
  python -c "import json; d=json.loads(open('gpurun_out/e9.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['clocks']['sm_mhz'], d['e2e']['value'])"
done; done
