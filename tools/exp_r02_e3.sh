set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_igemm.py tests/test_resnet.py tests/test_gpu_bench_shapes.py -x -q -m gpu > gpurun_out/e3_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/e3_tests.log
for prog in l1x1p l1x1r s3_1x1 s4_1x1 l3x3 stem l1x1; do
  timeout 300 python tools/ab_steps.py $prog 1024 4 - SB_IG_NOPIPE 2>&1 | tail -2
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 2 -c 1 \
      -o gpurun_out/e3b_l1x1p python tools/profile_steps.py l1x1p 1024 > gpurun_out/e3_ncu.log 2>&1; echo ncu rc=$?
