#!/bin/bash
# usage: tools/build_variant.sh <name> "<-D flags>"  -> build_variants/<name>/libckkt.so (experiments only)
set -e
cd "$(dirname "$0")/.."
mkdir -p build_variants/$1
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Xptxas -O3 --expt-relaxed-constexpr -I include"
nvcc $F $2 -c paper_2403_15913_b200/csrc/ckkt.cu -o build_variants/$1/ckkt.o
nvcc $F $2 -c paper_2403_15913_b200/csrc/model_eval.cu -o build_variants/$1/model_eval.o
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o build_variants/$1/libckkt.so build_variants/$1/ckkt.o \
  build_variants/$1/model_eval.o paper_2403_15913_b200/csrc/analysis.cpp.o -lcudart
echo build_variants/$1/libckkt.so
