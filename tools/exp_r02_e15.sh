set -u
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_conv.py -x -q -m gpu > gpurun_out/e15_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/e15_tests.log
SB_LIMB_TRACE=1 python bench.py --config c1_i32 --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | grep "limb CTA" | tail -3
for v in - SB_LIMB_NOSPLIT=1 -; do
  if [ "$v" = "-" ]; then timeout 300 python bench.py --config c1_i32 --steps 20 --no-cpu-baseline > gpurun_out/e13.json 2>/dev/null
  else env $v timeout 300 python bench.py --config c1_i32 --steps 20 --no-cpu-baseline > gpurun_out/e13.json 2>/dev/null; fi
  python -c "import json; d=json.loads(open('gpurun_out/e13.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['value'])"
done
