set -u
mkdir -p gpurun_out
for i in 1 2; do for v in default SB_IG_NOPIPE; do
  for prog in l1x1p s3_1x1; do
    if [ $v = default ]; then SB_PROFILE_STEPS=1 timeout 120 python tools/profile_steps.py $prog 1024 > /dev/null 2> gpurun_out/e2_${prog}_$v.txt
    else env $v=1 SB_PROFILE_STEPS=1 timeout 120 python tools/profile_steps.py $prog 1024 > /dev/null 2> gpurun_out/e2_${prog}_$v.txt; fi
    echo "$i $prog $v $(grep 'sb step' gpurun_out/e2_${prog}_$v.txt | awk '{print $4}' | tr '\n' ' ')"
  done
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 2 -c 1 \
      -o gpurun_out/e2_l1x1p python tools/profile_steps.py l1x1p 1024 > gpurun_out/e2_ncu.log 2>&1; echo ncu rc=$?
