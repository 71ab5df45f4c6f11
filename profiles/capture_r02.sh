#!/bin/bash
# Round-2 profiling capture (run on the GPU box via gpurun; writes into gpurun_out/).
#   1. dense int8 / tf32 peaks (tools/measure_peaks.py -> gpurun_out/r02_peaks.json)
#   2. per config: the plain run, then the ncu metric list of the same command for every
#      launch of the steps after the first (DRAM read/write, L2 write, tensor pipe, duration)
#      -> gpurun_out/ncu_<cfg>.csv (tools/ncu_traffic.py summarises them)
set -u
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed"
CFGS=${CFGS:-"c2 c3 c4a c4b c1 c1_i32 c5"}
# this library's kernels only (the runner's torch init kernels are not profiled or counted)
K="conv|gemm|reduce|pool|map_block|generic|fill_kernel|limb|tf32"
for cfg in $CFGS; do
  extra=""
  skip=2; cnt=4
  case $cfg in
    c5) extra="--batch 128"; skip=59; cnt=59;;
    c1_i32) skip=7; cnt=14;;
  esac
  CMD="python tools/run_config.py --config $cfg --steps 4 $extra"
  $CMD > gpurun_out/plain_$cfg.log 2>&1 && \
    ncu --metrics $M --clock-control none -k "regex:$K" -s $skip -c $cnt --csv --log-file gpurun_out/ncu_$cfg.csv $CMD \
      > gpurun_out/ncu_$cfg.log 2>&1
  echo "$cfg rc=$?"
done
# kernel families no BASELINE config isolates: the element-wise map kernel (config 3's epilogue
# unfused) and the windowed pool kernel (the ResNet stem max-pool)
for prog in ${PROGS:-"map pool"}; do
  CMD="python tools/run_config.py --program $prog --steps 4"
  $CMD > gpurun_out/plain_$prog.log 2>&1 && \
    ncu --metrics $M --clock-control none -k "regex:$K" -s 2 -c 2 --csv --log-file gpurun_out/ncu_$prog.csv $CMD \
      > gpurun_out/ncu_$prog.log 2>&1
  echo "$prog rc=$?"
done
