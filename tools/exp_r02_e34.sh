set -u
timeout 900 python -m pytest tests/test_gpu_igemm.py tests/test_resnet.py -x -q -m gpu > gpurun_out/e34_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/e34_tests.log
for prog in l1x1p l1x1r l1x1 l3x3 s2_1x1 s3_1x1 s4_1x1 s3_3x3 s3_1024 l24 l25 s2_3x3; do
  a=$(timeout 120 python tools/ab_steps.py $prog 1024 3 - 2>&1 | tail -1 | awk '{print $5}')
  b=$(SB_IG_STG4_ANY=1 timeout 120 python tools/ab_steps.py $prog 1024 3 - 2>&1 | tail -1 | awk '{print $5}')
  echo "$prog new $a old $b"
done
