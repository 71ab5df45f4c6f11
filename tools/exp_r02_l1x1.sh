# stage-1 1x1 layers: layouts (SB_IG_SHOW) and separate-process A/B of layout switches at b1024
set -u
for prog in l1x1p l1x1r l1x1 s2_1x1 l25; do
  SB_IG_SHOW=1 timeout 300 python tools/ab_steps.py $prog 1024 1 - 2>&1 | grep "igemm M" | head -1 | sed "s/^/$prog /"
done
for rep in 1 2; do
for prog in l1x1p l1x1; do
for v in - SB_IG_BN128 SB_IG_STG2 SB_IG_NOSPLIT SB_IG_KPB1 SB_IG_MT1 SB_IG_NOBRES; do
  if [ "$v" = "-" ]; then timeout 300 python tools/ab_steps.py $prog 1024 5 - 2>&1 | tail -1;
  else env $v=1 timeout 300 python tools/ab_steps.py $prog 1024 5 - 2>&1 | tail -1 | sed "s/ - / $v /"; fi
done; done; done
