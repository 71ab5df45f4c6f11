set -u
for prog in l3x3 s3_3x3 s3_1024 s4_1x1 s3_1x1; do
  for v in - SB_IG_KPB1=1 SB_IG_MT1=1 SB_IG_NOBRES=1 SB_IG_BN128=1; do
    if [ "$v" = "-" ]; then r=$(timeout 120 python tools/ab_steps.py $prog 1024 3 - 2>&1 | tail -1)
    else r=$(env $v timeout 120 python tools/ab_steps.py $prog 1024 3 - 2>&1 | tail -1); fi
    echo "$v $r"
  done
done
