#!/bin/bash
# Last round-2 status pass on one B200 (gpurun): GPU parity suite, smoke, every config's bench
# line, the C5 per-layer roofline table, the ncu launch list of the default bench command, and
# the per-config ncu launch metrics (profiles/capture_r02.sh).  Output: gpurun_out/fin/.
set -u
mkdir -p gpurun_out/fin
O=gpurun_out/fin
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$? | tee -a $O/rc.txt; tail -3 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$? | tee -a $O/rc.txt
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo bench rc=$? | tee -a $O/rc.txt
for c in c2 c3 c4a c4b c1 c1_i32; do
  timeout 600 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; echo $c rc=$? | tee -a $O/rc.txt
done
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo reference rc=$? | tee -a $O/rc.txt
timeout 600 python tools/c5_layers.py --batch 1024 > $O/layers_b1024.txt 2>&1; tail -1 $O/layers_b1024.txt
# launch list of the default bench command (cold, serialised per-launch times: shares, not absolutes)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:conv|gemm|reduce|pool|map_block|generic|fill_kernel|limb|fold" \
  -c 400 --csv --log-file $O/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_bench.log 2>&1
echo launches rc=$? | tee -a $O/rc.txt
CFGS="c2 c3 c4a c4b c1 c1_i32 c5" PROGS="map pool" bash profiles/capture_r02.sh > $O/capture.log 2>&1
mv gpurun_out/ncu_*.csv $O/ 2>/dev/null
for f in $O/bench_*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('ms_per_step'), d.get('value'), d.get('unit'), (d.get('roofline') or {}).get('frac'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('e2e') or {}).get('value'))" 2>&1; done | tee $O/summary.txt
