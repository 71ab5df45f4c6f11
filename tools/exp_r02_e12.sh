set -u
timeout 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_igemm.py tests/test_gpu_bench_shapes.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/e12_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/e12_tests.log
SB_TC_I8_EPI=1 timeout 900 python -m pytest tests/test_resnet.py tests/test_gpu_bench_shapes.py -x -q -m gpu > gpurun_out/e12_tests2.log 2>&1; echo tests-tci8 rc=$?; tail -1 gpurun_out/e12_tests2.log
for i in 1 2; do
for v in - SB_TC_I8_EPI=1; do
  if [ "$v" = "-" ]; then timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/e12.json 2>/dev/null
  else env $v timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/e12.json 2>/dev/null; fi
  python -c "import json; d=json.loads(open('gpurun_out/e12.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['clocks']['sm_mhz'])"
done; done
