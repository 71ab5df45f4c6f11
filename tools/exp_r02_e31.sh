set -u
for prog in s3_1x1 s2_1x1; do
  for v in - SB_IG_BN128=1 SB_IG_STG2=1; do
    if [ "$v" = "-" ]; then r=$(timeout 120 python tools/ab_steps.py $prog 1024 3 - 2>&1 | tail -1)
    else r=$(env $v timeout 120 python tools/ab_steps.py $prog 1024 3 - 2>&1 | tail -1); fi
    echo "$v $r"
  done
done
SB_LIBRARY=$PWD/paper_1903_06498_b200/libstripe_b200_trace.so timeout 120 python tools/profile_steps.py s3_1x1 1024 > /dev/null 2> gpurun_out/e31t.txt
