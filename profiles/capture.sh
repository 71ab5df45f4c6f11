#!/bin/bash
# Round profiling capture (run on the GPU box via gpurun; writes into gpurun_out/).
#   1. the bench line (no profiler)
#   2. the ncu launch list of the same command (cold-cache, serialised per-launch times)
#   3. one `ncu --set full` capture of the conv kernel
set -u
mkdir -p gpurun_out
python bench.py --steps 50 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
CMD="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD \
  > gpurun_out/ncu_launch.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:conv_i8 -s 3 -c 1 -o gpurun_out/prof_conv $CMD \
  > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
cat gpurun_out/bench.json
