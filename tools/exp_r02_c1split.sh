set -u
python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/gemm_tests.log 2>&1; echo EXIT $? >> gpurun_out/gemm_tests.log
for rep in 1 2; do
for v in split nosplit; do
  if [ $v = nosplit ]; then export SB_GEMM_NOSPLIT=1; else unset SB_GEMM_NOSPLIT; fi
  python bench.py --config c1 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['ms_per_step']*1000, 'us', d['roofline']['kernel_ms_per_step']*1000, 'us kernel', d['value'])" >> gpurun_out/c1ab.log 2>&1
done; done
unset SB_GEMM_NOSPLIT
