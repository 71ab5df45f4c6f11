set -u
for prog in l1x1r s2_1x1 s3_1x1 s4_1x1; do
  for i in 1 2; do
    timeout 120 python tools/ab_steps.py $prog 1024 3 - 2>&1 | tail -1
    SB_IG_RESEPI=1 timeout 120 python tools/ab_steps.py $prog 1024 3 - 2>&1 | tail -1 | sed 's/^/RESEPI /'
  done
done
