#!/bin/bash
# Steady-state DRAM traffic per launch (write-back counted): like capture_r02.sh but with
# `--cache-control none`, profiling launches after the input/output set rotation has cycled
# (the working set is > 3x L2), so the dirty outputs of earlier launches are written back
# inside the profiled ones -- per launch, DRAM write then approximates the bytes a launch
# really stores.  -> gpurun_out/ncuw_<cfg>.csv (tools/ncu_traffic.py summarises them)
set -u
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
K="conv|gemm|reduce|pool|map_block|generic|fill_kernel|limb|tf32"
CFGS=${CFGS:-"c2 c3 c4a c4b c1 c1_i32"}
for cfg in $CFGS; do
  skip=12; cnt=6
  case $cfg in c1_i32) skip=30; cnt=12;; esac
  CMD="python tools/run_config.py --config $cfg --steps 24"
  ncu --metrics $M --clock-control none --cache-control none -k "regex:$K" -s $skip -c $cnt --csv \
      --log-file gpurun_out/ncuw_$cfg.csv $CMD > gpurun_out/ncuw_$cfg.log 2>&1
  echo "$cfg rc=$?"
done
