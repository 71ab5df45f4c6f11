# resident-filter conv: two staging buffers per epilogue group (was opt-in SB_CONV_STG4, now the default; SB_CONV_STG2 restores one per group)
set -u
SB_CONV_STG4=1 python -m pytest tests/test_gpu_conv.py tests/test_gpu_bench_shapes.py tests/test_pipeline_programs.py -q -x -k "not c5" > gpurun_out/stg4_tests.log 2>&1; echo EXIT $? >> gpurun_out/stg4_tests.log
for rep in 1 2; do
for v in base stg4; do
  for c in c2 c3; do
    if [ $v = stg4 ]; then export SB_CONV_STG4=1; else unset SB_CONV_STG4; fi
    python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $c', d['ms_per_step']*1000, 'us', d['roofline']['frac'], 'kernel', d['roofline'].get('kernel_ms_per_step'))" >> gpurun_out/stg4_ab.log 2>&1
  done
done; done
unset SB_CONV_STG4
