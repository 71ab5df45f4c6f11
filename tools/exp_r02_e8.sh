set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_igemm.py tests/test_resnet.py tests/test_gpu_bench_shapes.py -x -q -m gpu > gpurun_out/e8_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/e8_tests.log
for prog in s2_1x1 s3_1x1 l11 s3_3x3; do
  for i in 1 2; do
    timeout 120 python tools/ab_steps.py $prog 1024 3 - 2>&1 | tail -1
    SB_IG_NONSTAT=1 timeout 120 python tools/ab_steps.py $prog 1024 3 - 2>&1 | tail -1 | sed 's/^/NONSTAT /'
  done
done
for prog in s2_1x1 s3_1x1; do
SB_LIBRARY=$PWD/paper_1903_06498_b200/libstripe_b200_trace.so timeout 120 python tools/profile_steps.py $prog 1024 > /dev/null 2> gpurun_out/e8t_$prog.txt
done
