set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_igemm.py -x -q -m gpu -k "band" > gpurun_out/e5_band.log 2>&1; echo band rc=$?; tail -15 gpurun_out/e5_band.log
timeout 900 python -m pytest tests/test_gpu_igemm.py tests/test_resnet.py tests/test_gpu_bench_shapes.py -x -q -m gpu > gpurun_out/e5_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/e5_tests.log
for i in 1 2; do
timeout 120 python tools/ab_steps.py stem 1024 3 - 2>&1 | tail -1
SB_NO_BAND=1 timeout 120 python tools/ab_steps.py stem 1024 3 - 2>&1 | tail -1
done
