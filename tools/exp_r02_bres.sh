# A/B of the resident-filter cap (SB_IG_BRES_KB) on the 1x1 layers whose filter slices exceed
# 96 KB: separate processes (the prepare cache keys on the plan), interleaved twice.
set -u
for rep in 1 2; do
for prog in s3_1024 l44 l43 l47 s3_1x1; do
for cap in 96 128 160; do
  SB_IG_BRES_KB=$cap timeout 300 python tools/ab_steps.py $prog 1024 5 - 2>&1 | sed "s/^/cap=$cap /" | tail -1
done; done; done
