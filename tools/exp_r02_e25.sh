set -u
timeout 900 python -m pytest tests/test_gpu_igemm.py tests/test_resnet.py tests/test_gpu_bench_shapes.py -x -q -m gpu > gpurun_out/e25_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/e25_tests.log
for prog in l1x1p l1x1r s4_1x1 s3_1x1 s2_1x1 l25; do timeout 120 python tools/ab_steps.py $prog 1024 3 - 2>&1 | tail -1; done
timeout 300 python tools/c5_layers.py --batch 1024 > gpurun_out/e25_layers.txt 2>&1; tail -1 gpurun_out/e25_layers.txt
timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/e25.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/e25.json').read().strip().splitlines()[-1]); print('C5', d['ms_per_step'], d['clocks']['sm_mhz'])"
