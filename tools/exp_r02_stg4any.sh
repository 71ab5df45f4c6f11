# im2col conv: the second staging buffer per epilogue group forced wherever it fits
# (SB_IG_STG4_ANY) vs the planner's rule, separate processes, b1024
set -u
for prog in l1x1r s2_1x1 s3_1x1 s4_1x1 l3x3 s2_3x3 s3_3x3 s4_3x3 l24 l25 l11 l44 l47 s3_1024 l1x1; do
  a=$(timeout 300 python tools/ab_steps.py $prog 1024 5 - 2>&1 | tail -1 | awk '{print $5}')
  b=$(SB_IG_STG4_ANY=1 timeout 300 python tools/ab_steps.py $prog 1024 5 - 2>&1 | tail -1 | awk '{print $5}')
  s=$(SB_IG_SHOW=1 SB_IG_STG4_ANY=1 timeout 300 python tools/ab_steps.py $prog 1024 1 - 2>&1 | grep -o "stages=[0-9]* .*stg4=[0-9]" | head -1)
  echo "$prog base $a stg4_any $b ($s)"
done
