set -u
timeout 900 python -m pytest tests/test_gpu_igemm.py tests/test_gpu_conv.py tests/test_gpu_bench_shapes.py -x -q -m gpu > gpurun_out/e64_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/e64_tests.log
for i in 1 2; do
  timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/e64.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/e64.json').read().strip().splitlines()[-1]); print('C5', d['ms_per_step'], d['clocks']['sm_mhz'])"
done
timeout 300 python tools/c5_layers.py --batch 1024 > gpurun_out/e64_layers.txt 2>&1; tail -1 gpurun_out/e64_layers.txt
