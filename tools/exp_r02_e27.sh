set -u
for b in 128 256 512; do
timeout 300 python bench.py --batch $b --steps 10 --no-cpu-baseline > gpurun_out/e27.json 2>gpurun_out/e27.err; python -c "import json; d=json.loads(open('gpurun_out/e27.json').read().strip().splitlines()[-1]); print('C5 b$b', d['ms_per_step'], d['value'], d['clocks']['sm_mhz'], d['e2e']['dropin']['value'])" || tail -3 gpurun_out/e27.err
done
