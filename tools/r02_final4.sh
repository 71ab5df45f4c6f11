#!/bin/bash
# After the conv_tc staging change: whole GPU suite, smoke, C2/C3/C5 lines
set -u
O=gpurun_out/fin4
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$? | tee -a $O/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$? | tee -a $O/rc.txt
for c in c2 c3; do
  timeout 600 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; echo $c rc=$? | tee -a $O/rc.txt
done
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo c5 rc=$? | tee -a $O/rc.txt
for f in $O/bench_*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); e=d.get('e2e') or {}; print('$f', d.get('ms_per_step'), d.get('value'), d.get('unit'), (d.get('roofline') or {}).get('frac'), (d.get('clocks') or {}).get('sm_mhz'), 'e2e', e.get('value'), 'dropin', (e.get('dropin') or {}).get('value'))" 2>&1; done | tee $O/summary.txt
