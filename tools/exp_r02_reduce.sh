# short-reduction kernel (32-bit indexing, all loads in flight) vs the table-driven kernel
set -u
python -m pytest tests/test_gpu_map.py tests/test_gpu_bench_shapes.py -q -k "not c5 and not c3" > gpurun_out/reduce_tests.log 2>&1; echo EXIT $? >> gpurun_out/reduce_tests.log
python tools/ab_steps.py c4a 128 10 - SB_REDUCE_LONG > gpurun_out/reduce_ab.log 2>&1
python tools/ab_steps.py c5 1024 3 - SB_REDUCE_LONG 2>&1 | tail -2 | cut -c1-200 >> gpurun_out/reduce_ab.log
for c in c4a c4b; do python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['value'], d['roofline']['frac'])" >> gpurun_out/reduce_ab.log; done
