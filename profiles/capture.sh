#!/bin/bash
# Round profiling capture (run on the GPU box via gpurun; writes into gpurun_out/).
#   1. the bench lines (no profiler): config 2 (default) and config 5
#   2. the ncu launch lists of the same commands (cold-cache, serialised per-launch times)
#   3. `ncu --set full` captures: the config-2 conv kernel, the config-5 stem and a
#      stage-1 3x3 im2col conv (tools/profile_steps.py programs)
set -u
mkdir -p gpurun_out
python bench.py --steps 50 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --config c5 --steps 20 --warmup 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
C2="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
C5="python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline"
$C2 > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $C2 \
  > gpurun_out/ncu_launch.log 2>&1
$C5 > gpurun_out/plain_c5.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c5.csv $C5 \
  > gpurun_out/ncu_launch_c5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_i8 -s 3 -c 1 -o gpurun_out/prof_conv $C2 \
  > gpurun_out/ncu_full.log 2>&1
for prog in stem l3x3; do
  python tools/profile_steps.py $prog 128 > /dev/null 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 1 -c 1 \
      -o gpurun_out/prof_$prog python tools/profile_steps.py $prog 128 > gpurun_out/ncu_$prog.log 2>&1
done
tail -2 gpurun_out/ncu_full.log
cut -c1-300 gpurun_out/bench.json gpurun_out/bench_c5.json
