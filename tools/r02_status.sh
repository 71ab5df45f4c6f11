set -u
# round-2 status pass: GPU parity, smoke, default bench line, per-config lines, C5 per-layer table
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/s_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/s_smoke.log
timeout 600 python bench.py > gpurun_out/s_bench_c5.json 2> gpurun_out/s_bench_c5.err; echo bench rc=$?
for c in c2 c3 c4a c4b c1 c1_i32; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/s_bench_$c.json 2> gpurun_out/s_bench_$c.err; echo $c rc=$?
done
timeout 300 python tools/c5_layers.py --batch 1024 > gpurun_out/s_layers.txt 2>&1; tail -1 gpurun_out/s_layers.txt
for f in gpurun_out/s_bench_*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['value'], d['unit'], d['roofline'].get('frac'), d['clocks'].get('sm_mhz'))"; done
