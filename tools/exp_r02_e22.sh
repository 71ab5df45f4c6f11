set -u
timeout 900 python -m pytest tests/test_gpu_igemm.py -x -q -m gpu -k "strip" > gpurun_out/e22_strip.log 2>&1; echo strip rc=$?; tail -15 gpurun_out/e22_strip.log
timeout 900 python -m pytest tests/test_gpu_igemm.py tests/test_resnet.py tests/test_gpu_bench_shapes.py -x -q -m gpu > gpurun_out/e22_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/e22_tests.log
for i in 1 2; do
timeout 120 python tools/ab_steps.py l3x3 1024 3 - 2>&1 | tail -1
SB_IG_NOSTRIP=1 timeout 120 python tools/ab_steps.py l3x3 1024 3 - 2>&1 | tail -1 | sed 's/^/NOSTRIP /'
done
