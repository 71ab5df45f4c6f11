set -u
mkdir -p gpurun_out
export SB_PROFILE_STEPS=1
timeout 120 python tools/profile_steps.py stem 1024 > /dev/null 2> gpurun_out/e6_steps.txt; grep "sb step" gpurun_out/e6_steps.txt | tail -4
SB_LIBRARY=$PWD/paper_1903_06498_b200/libstripe_b200_trace.so timeout 120 python tools/profile_steps.py stem 1024 > /dev/null 2> gpurun_out/e6t_stem.txt
unset SB_PROFILE_STEPS
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 20 --csv python tools/profile_steps.py stem 1024 > gpurun_out/e6_launches.csv 2>&1; echo ncu1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 1 -c 1 -o gpurun_out/e6_stem python tools/profile_steps.py stem 1024 > gpurun_out/e6_ncu.log 2>&1; echo ncu rc=$?
