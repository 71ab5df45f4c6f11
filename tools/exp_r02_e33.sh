set -u
for v in - SB_IG_STG2=1; do
  if [ "$v" = "-" ]; then r=$(timeout 120 python tools/ab_steps.py s4_1x1 1024 3 - 2>&1 | tail -1)
  else r=$(env $v timeout 120 python tools/ab_steps.py s4_1x1 1024 3 - 2>&1 | tail -1); fi
  echo "$v $r"
done
SB_LIBRARY=$PWD/paper_1903_06498_b200/libstripe_b200_trace.so timeout 120 python tools/profile_steps.py s4_1x1 1024 2>&1 >/dev/null | grep "igemm M=" | tail -1
SB_IG_STG2=1 SB_LIBRARY=$PWD/paper_1903_06498_b200/libstripe_b200_trace.so timeout 120 python tools/profile_steps.py s4_1x1 1024 2>&1 >/dev/null | grep "igemm M=" | tail -1
