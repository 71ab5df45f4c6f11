#!/bin/bash
# Experiment builds of the im2col conv kernel with compile-time knock-out bits (conv_igemm.cu
# EXPB / EPI_EXP): scratch/libstripe_b200_e<N>.so for each N, every other object from build/.
#   bash tools/exp_build.sh 258 514 ...   then   SB_LIBRARY=$PWD/scratch/libstripe_b200_e258.so ...
set -e
cd "$(dirname "$0")/../paper_1903_06498_b200"
make -s -j8 libstripe_b200.so >/dev/null
NV="/usr/local/cuda/bin/nvcc -ccbin /usr/bin/g++ -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr"
for n in "$@"; do
  $NV -DSB_EXP_CONST=$n -Xptxas -v -c csrc/kernels/conv_igemm.cu -o ../scratch/cu_conv_igemm_e$n.o 2> ../scratch/e$n.ptxas.log &
done
wait
for n in "$@"; do
  grep -A3 conv_igemm_i8_kernel ../scratch/e$n.ptxas.log | grep -o "[0-9]* bytes spill stores" | head -1 | sed "s/^/e$n: /"
  objs=$(ls build/*.o | grep -v cu_conv_igemm.o)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../scratch/libstripe_b200_e$n.so $objs ../scratch/cu_conv_igemm_e$n.o -cudart static -Xlinker -z,defs -lpthread -ldl -lrt
done
