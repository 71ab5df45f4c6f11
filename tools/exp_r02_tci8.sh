# stage-1 3x3 convs (56x56x64->64, i8 out) on the resident-filter kernel (SB_TC_I8_EPI) now that
# it double-buffers its staging per epilogue group; separate processes (routing is planned once)
set -u
SB_TC_I8_EPI=1 python -m pytest tests/test_gpu_conv.py tests/test_resnet.py -q -x > gpurun_out/tci8_tests.log 2>&1; echo EXIT $? >> gpurun_out/tci8_tests.log
for rep in 1 2; do
  echo "igemm  $(timeout 300 python tools/ab_steps.py l3x3 1024 5 - 2>&1 | tail -1 | cut -c1-80)"
  echo "tc_i8  $(SB_TC_I8_EPI=1 timeout 300 python tools/ab_steps.py l3x3 1024 5 - 2>&1 | tail -1 | cut -c1-80)"
  echo "tc_i8_stg2  $(SB_CONV_STG2=1 SB_TC_I8_EPI=1 timeout 300 python tools/ab_steps.py l3x3 1024 5 - 2>&1 | tail -1 | cut -c1-80)"
done
echo "c5 igemm $(timeout 600 python tools/ab_steps.py c5 1024 3 - 2>&1 | tail -1 | cut -c1-60)"
echo "c5 tc_i8 $(SB_TC_I8_EPI=1 timeout 600 python tools/ab_steps.py c5 1024 3 - 2>&1 | tail -1 | cut -c1-60)"
echo "c5 bench igemm $(timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-200)"
echo "c5 bench tc_i8 $(SB_TC_I8_EPI=1 timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-200)"
