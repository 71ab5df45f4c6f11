set -u
timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q -m gpu > gpurun_out/e13_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/e13_tests.log
for i in 1 2; do for v in - SB_LIMB_UNFUSED=1 SB_LIMB_NOSPLIT=1; do
  if [ "$v" = "-" ]; then timeout 300 python bench.py --config c1_i32 --steps 20 --no-cpu-baseline > gpurun_out/e13.json 2>/dev/null
  else env $v timeout 300 python bench.py --config c1_i32 --steps 20 --no-cpu-baseline > gpurun_out/e13.json 2>/dev/null; fi
  python -c "import json; d=json.loads(open('gpurun_out/e13.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['value'], d['roofline'].get('isolated'))"
done; done
