set -u
mkdir -p gpurun_out
python -m pytest tests/test_gpu_igemm.py tests/test_resnet.py tests/test_gpu_bench_shapes.py -x -q -m gpu > gpurun_out/e4_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/e4_tests.log
for v in default SB_IG_STG2; do
  for prog in l1x1p s3_1x1 l1x1r s4_1x1 l3x3; do
    if [ $v = default ]; then SB_PROFILE_STEPS=1 python tools/profile_steps.py $prog 1024 > /dev/null 2> gpurun_out/e4_${prog}_$v.txt
    else env $v=1 SB_PROFILE_STEPS=1 python tools/profile_steps.py $prog 1024 > /dev/null 2> gpurun_out/e4_${prog}_$v.txt; fi
    echo "$prog $v $(tail -1 gpurun_out/e4_${prog}_$v.txt)"
  done
done
python bench.py --steps 10 --no-cpu-baseline > gpurun_out/e4_c5.json 2>&1
SB_IG_STG2=1 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/e4_c5_stg2.json 2>&1
for f in gpurun_out/e4_c5*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['clocks']['sm_mhz'])"; done
python tools/c5_layers.py --batch 1024 > gpurun_out/e4_layers.txt 2>&1; tail -1 gpurun_out/e4_layers.txt
