# band stem: second staging buffer per epilogue group (SB_IG_BAND_STG4; shortens the ring)
set -u
SB_IG_BAND_STG4=1 python -m pytest tests/test_gpu_igemm.py tests/test_resnet.py -q -x > gpurun_out/bstg4_tests.log 2>&1; echo EXIT $? >> gpurun_out/bstg4_tests.log
for rep in 1 2; do
  echo "base   $(SB_IG_SHOW=1 timeout 300 python tools/ab_steps.py stem 1024 5 - 2>&1 | grep -E 'igemm M|total' | tr '\n' ' ' | cut -c1-400)"
  echo "stg4   $(SB_IG_SHOW=1 SB_IG_BAND_STG4=1 timeout 300 python tools/ab_steps.py stem 1024 5 - 2>&1 | grep -E 'igemm M|total' | tr '\n' ' ' | cut -c1-400)"
done
