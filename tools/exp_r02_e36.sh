set -u
for prog in l3x3 s3_1x1 s4_1x1; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 1 -c 1 -o gpurun_out/e36_$prog python tools/profile_steps.py $prog 1024 > /dev/null 2>&1; echo $prog rc=$?
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_limb -s 2 -c 1 -o gpurun_out/e36_limb python bench.py --config c1_i32 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo limb rc=$?
