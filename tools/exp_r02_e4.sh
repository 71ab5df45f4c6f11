set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/e4_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/e4_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/e4_c5.json 2> gpurun_out/e4_c5.err; echo bench rc=$?
python -c "import json; d=json.loads(open('gpurun_out/e4_c5.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['clocks'])"
timeout 300 python tools/c5_layers.py --batch 1024 > gpurun_out/e4_layers.txt 2>&1; tail -1 gpurun_out/e4_layers.txt
