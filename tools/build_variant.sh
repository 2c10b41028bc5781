#!/bin/bash
# Build an experimental variant of libaco_gpu.so with extra -D flags:
#   tools/build_variant.sh NAME -DACO_TIMING=1 ...  -> paper_1101_2678_b200/libaco_gpu_NAME.so
set -e
cd "$(dirname "$0")/../paper_1101_2678_b200/csrc"
name=$1; shift
make -s _build/host_model.o
mkdir -p _build/$name
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false \
  -Xcompiler -fPIC,-ffp-contract=off "$@" -c aco_gpu.cu -o _build/$name/aco_gpu.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
  -o ../libaco_gpu_$name.so _build/$name/aco_gpu.o _build/host_model.o -ldl -lpthread
echo "built paper_1101_2678_b200/libaco_gpu_$name.so"
