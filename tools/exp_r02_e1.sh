set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_igemm.py tests/test_resnet.py tests/test_gpu_bench_shapes.py -x -q -m gpu > gpurun_out/e1_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/e1_tests.log
for v in default SB_IG_NOPIPE; do
  for prog in l1x1p l1x1r l3x3 stem s3_1x1 l1x1 s4_1x1; do
    if [ $v = default ]; then SB_PROFILE_STEPS=1 timeout 120 python tools/profile_steps.py $prog 1024 > /dev/null 2> gpurun_out/e1_${prog}_$v.txt
    else env $v=1 SB_PROFILE_STEPS=1 timeout 120 python tools/profile_steps.py $prog 1024 > /dev/null 2> gpurun_out/e1_${prog}_$v.txt; fi
    echo "$prog $v $(tail -1 gpurun_out/e1_${prog}_$v.txt)"
  done
done
timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/e1_c5.json 2>&1
SB_IG_NOPIPE=1 timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/e1_c5_nopipe.json 2>&1
for f in gpurun_out/e1_c5*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['clocks']['sm_mhz'])"; done
export SB_LIBRARY=$PWD/paper_1903_06498_b200/libstripe_b200_trace.so
for prog in l1x1p l3x3; do
  timeout 120 python tools/profile_steps.py $prog 1024 > /dev/null 2> gpurun_out/e1t_$prog.txt; echo $prog rc=$?
done
