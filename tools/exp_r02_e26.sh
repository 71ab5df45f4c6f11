set -u
timeout 900 python -m pytest tests/test_gpu_pool.py tests/test_resnet.py tests/test_gpu_bench_shapes.py -x -q -m gpu > gpurun_out/e26_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/e26_tests.log
timeout 300 python tools/ab_steps.py pool 1024 4 - SB_POOL_SINGLE 2>&1 | tail -2
