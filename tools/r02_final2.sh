#!/bin/bash
# Re-check after the last kernel changes (reduce short/unrolled windows, 128x256 GEMM tiles):
# the whole GPU suite, smoke, and the bench lines those kernels touch. Output: gpurun_out/fin2/.
set -u
O=gpurun_out/fin2
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$? | tee -a $O/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$? | tee -a $O/rc.txt
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo bench rc=$? | tee -a $O/rc.txt
for c in c4a c4b c1 c1_i32; do
  timeout 600 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; echo $c rc=$? | tee -a $O/rc.txt
done
for f in $O/bench_*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('ms_per_step'), d.get('value'), d.get('unit'), (d.get('roofline') or {}).get('frac'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('e2e') or {}).get('value'))" 2>&1; done | tee $O/summary.txt
