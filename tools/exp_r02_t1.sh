set -u
mkdir -p gpurun_out
export SB_LIBRARY=$PWD/paper_1903_06498_b200/libstripe_b200_trace.so
for prog in l1x1p l1x1r l3x3 stem s3_1x1 l1x1; do
  timeout 120 python tools/profile_steps.py $prog 1024 > /dev/null 2> gpurun_out/t1_$prog.txt; echo $prog rc=$?
done
