set -u
timeout 900 python -m pytest tests/test_gpu_igemm.py tests/test_resnet.py tests/test_gpu_bench_shapes.py -x -q -m gpu > gpurun_out/e18_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/e18_tests.log
for prog in s4_1x1 l24 l25 s3_1x1 s2_1x1; do
  for v in - SB_IG_NSTAT8=1; do
    if [ "$v" = "-" ]; then r=$(timeout 120 python tools/ab_steps.py $prog 1024 3 - 2>&1 | tail -1)
    else r=$(env $v timeout 120 python tools/ab_steps.py $prog 1024 3 - 2>&1 | tail -1); fi
    echo "$v $r"
  done
done
for i in 1 2; do for v in - SB_IG_NSTAT8=1; do
  if [ "$v" = "-" ]; then timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/e18.json 2>/dev/null
  else env $v timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/e18.json 2>/dev/null; fi
  python -c "import json; d=json.loads(open('gpurun_out/e18.json').read().strip().splitlines()[-1]); print('C5 $v', d['ms_per_step'], d['clocks']['sm_mhz'])"
done; done
