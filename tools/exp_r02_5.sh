set -u
mkdir -p gpurun_out
python -m pytest tests/test_gpu_bench_shapes.py tests/test_gpu_pdl.py tests/test_pipeline_programs.py tests/test_gpu_conv.py -x -q -m gpu > gpurun_out/e5_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/e5_tests.log
SB_IG_STG2=1 python tools/c5_layers.py --batch 1024 > gpurun_out/e5_layers_stg2.txt 2>&1; tail -1 gpurun_out/e5_layers_stg2.txt
python tools/c5_layers.py --batch 1024 > gpurun_out/e5_layers_stg4.txt 2>&1; tail -1 gpurun_out/e5_layers_stg4.txt
