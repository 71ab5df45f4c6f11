set -u
mkdir -p gpurun_out
SB_TC_I8_EPI=1 SB_PROFILE_STEPS=1 python tools/profile_steps.py l3x3 1024 > /dev/null 2> gpurun_out/e2_l3x3_tci8.txt
SB_TC_I8_EPI=1 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/e2_c5_tci8.json 2>&1
SB_TC_I8_EPI=1 python tools/c5_layers.py --batch 1024 > gpurun_out/e2_c5_layers_tci8.txt 2>&1
python -c "import json; d=json.loads(open('gpurun_out/e2_c5_tci8.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks'])"
tail -3 gpurun_out/e2_l3x3_tci8.txt
grep -E "L0[369]|L1[69]|L22|TOTAL" gpurun_out/e2_c5_layers_tci8.txt
