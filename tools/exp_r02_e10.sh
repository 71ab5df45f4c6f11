set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_igemm.py tests/test_gpu_bench_shapes.py tests/test_golden.py -x -q -m gpu > gpurun_out/e10_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/e10_tests.log
for c in c2 c3; do for v in - SB_TC_NOPIPE=1; do
  if [ "$v" = "-" ]; then timeout 300 python bench.py --config $c --steps 20 --no-cpu-baseline > gpurun_out/e10.json 2>/dev/null
  else env $v timeout 300 python bench.py --config $c --steps 20 --no-cpu-baseline > gpurun_out/e10.json 2>/dev/null; fi
  python -c "import json; d=json.loads(open('gpurun_out/e10.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$c $v', d['ms_per_step'], r['frac'], r.get('isolated'))"
done; done
for i in 1 2; do
timeout 120 python tools/ab_steps.py l3x3 1024 3 - SB_TC_NOPIPE 2>&1 | tail -2
SB_TC_I8_EPI=1 timeout 120 python tools/ab_steps.py l3x3 1024 3 - SB_TC_NOPIPE 2>&1 | tail -2 | sed 's/^/TC /'
done
