set -u
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"limb|gemm" -c 12 --csv python bench.py --config c1_i32 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/e14_launches.csv 2>/dev/null; echo ncu rc=$?

timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q -m gpu > gpurun_out/e14_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/e14_tests.log
for v in - SB_LIMB_NOSPLIT=1 -; do
  if [ "$v" = "-" ]; then timeout 300 python bench.py --config c1_i32 --steps 20 --no-cpu-baseline > gpurun_out/e13.json 2>/dev/null
  else env $v timeout 300 python bench.py --config c1_i32 --steps 20 --no-cpu-baseline > gpurun_out/e13.json 2>/dev/null; fi
  python -c "import json; d=json.loads(open('gpurun_out/e13.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['value'])"
done
