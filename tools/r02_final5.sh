#!/bin/bash
# Last check of the committed tree: whole GPU suite, smoke, default bench line, reference arm
set -u
O=gpurun_out/fin5
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$? | tee -a $O/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$? | tee -a $O/rc.txt
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo c5 rc=$? | tee -a $O/rc.txt
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo ref rc=$? | tee -a $O/rc.txt
