set -u
mkdir -p gpurun_out
python bench.py --steps 10 --no-cpu-baseline > gpurun_out/e1_default.json 2>&1
SB_LANES=1 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/e1_lanes1.json 2>&1
SB_LANES=2 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/e1_lanes2.json 2>&1
for v in default SB_FOLD_OVERLAP SB_NO_FOLD; do
  if [ $v = default ]; then env SB_PROFILE_STEPS=1 python tools/profile_steps.py stem 1024 > /dev/null 2> gpurun_out/e1_stem_$v.txt
  else env $v=1 SB_PROFILE_STEPS=1 python tools/profile_steps.py stem 1024 > /dev/null 2> gpurun_out/e1_stem_$v.txt; fi
done
for v in default SB_IG_MT1 SB_IG_KPB1 SB_IG_NOBRES SB_IG_KPB3 SB_IG_NOSPLIT; do
  if [ $v = default ]; then env SB_PROFILE_STEPS=1 python tools/profile_steps.py l3x3 1024 > /dev/null 2> gpurun_out/e1_l3x3_$v.txt
  else env $v=1 SB_PROFILE_STEPS=1 python tools/profile_steps.py l3x3 1024 > /dev/null 2> gpurun_out/e1_l3x3_$v.txt; fi
done
for f in gpurun_out/e1_*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks'])"; done
for f in gpurun_out/e1_stem_* gpurun_out/e1_l3x3_*; do echo $f; tail -3 $f; done
