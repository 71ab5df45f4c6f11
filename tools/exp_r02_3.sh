set -u
mkdir -p gpurun_out
for prog in l3x3 stem l1x1p s3_1x1; do
  python tools/profile_steps.py $prog 1024 > /dev/null 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 2 -c 1 \
      -o gpurun_out/r02_prof_$prog python tools/profile_steps.py $prog 1024 > gpurun_out/ncu_full_$prog.log 2>&1
  echo $prog rc=$?
done
