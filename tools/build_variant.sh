#!/bin/bash
# Build a variant of libharvest_b200.so with extra -D flags into build/NAME/
# (select it with HARVEST_B200_LIB=build/NAME/libharvest_b200.so).
#   bash tools/build_variant.sh NAME -DHV_FFN_TMA=0 ...
NAME=$1; shift
mkdir -p build/$NAME
C=paper_2602_00328_b200/csrc
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-fvisibility=hidden \
  -shared -cudart static -I include "$@" -o build/$NAME/libharvest_b200.so \
  $C/hv_kernels.cu $C/hv_ffn.cu $C/hv_attn.cu $C/hv_moe.cu $C/hv_pool.cpp $C/hv_segalloc.cpp $C/hv_place.cpp -ldl -lrt -lpthread
