#!/bin/bash
# Build a libgfcuda variant with extra compile-time switches for A/B timing:
#   tools/build_variant.sh NAME "-DGF_SPLIT_MV=1 -DGF_HOLE_ILP=4"
# -> paper_2506_23775_b200/variants/libgfcuda_NAME.so (select with GF_LIB_PATH)
set -e
cd "$(dirname "$0")/../paper_2506_23775_b200/csrc"
NAME=$1; shift
OUT=../variants; mkdir -p $OUT
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -cudart static"
T=$(mktemp -d)
for s in gf_ops gf_target gf_hessian; do nvcc $F -c -o $T/$s.o $s.cu & done
nvcc $F $@ -c -o $T/gf_engine.o gf_engine.cu &
wait
nvcc $F -shared -o $OUT/libgfcuda_$NAME.so $T/*.o
rm -rf $T
