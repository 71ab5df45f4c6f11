# stage-3/4 layers: layouts (SB_IG_SHOW) and separate-process A/B of layout switches at b1024
set -u
for prog in ${SHOW_PROGS:-}; do
  SB_IG_SHOW=1 timeout 300 python tools/ab_steps.py $prog 1024 1 - 2>&1 | grep "igemm M" | head -1 | sed "s/^/$prog /"
done
for prog in s4_1x1 s4_3x3 s3_3x3 s3_1x1; do
for v in - SB_IG_BN128 SB_IG_STG2 SB_IG_KPB1 SB_IG_KPB3 SB_IG_NONSTAT SB_IG_NSTAT8 SB_IG_NOBRES; do
  if [ "$v" = "-" ]; then timeout 300 python tools/ab_steps.py $prog 1024 5 - 2>&1 | tail -1;
  else case $v in *=*) kv=$v;; *) kv=$v=1;; esac; env $kv timeout 300 python tools/ab_steps.py $prog 1024 5 - 2>&1 | tail -1 | sed "s/ - / $v /"; fi
done; done
