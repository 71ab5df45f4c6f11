# m-tile traversal reversal in the im2col conv (SB_IG_REV): parity with every launch reversed
# and alternating, then C5 per-step times with the three settings interleaved in one process
set -u
SB_IG_REV=1 python -m pytest tests/test_gpu_igemm.py tests/test_resnet.py tests/test_gpu_bench_shapes.py -q -x > gpurun_out/rev_tests.log 2>&1; echo EXIT1 $? >> gpurun_out/rev_tests.log
SB_IG_REV=alt python -m pytest tests/test_gpu_igemm.py tests/test_resnet.py tests/test_gpu_bench_shapes.py -q -x >> gpurun_out/rev_tests.log 2>&1; echo EXITalt $? >> gpurun_out/rev_tests.log
python tools/ab_steps.py c5 1024 4 - SB_IG_REV=alt SB_IG_REV=1 > gpurun_out/rev_ab.log 2>&1
