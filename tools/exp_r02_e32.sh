set -u
timeout 900 python -m pytest tests/test_gpu_igemm.py tests/test_resnet.py tests/test_gpu_bench_shapes.py -x -q -m gpu > gpurun_out/e32_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/e32_tests.log
for prog in l1x1r s2_1x1 s3_1x1 s4_1x1; do timeout 120 python tools/ab_steps.py $prog 1024 3 - 2>&1 | tail -1; done
