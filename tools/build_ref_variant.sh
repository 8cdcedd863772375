#!/bin/bash
# usage: tools/build_ref_variant.sh <name> <git-ref> ["<-D flags>"]  -> build_variants/<name>/libckkt.so
set -e -o pipefail
cd "$(dirname "$0")/.."
d=build_variants/src_$1
rm -rf $d; mkdir -p $d/x/csrc $d/include build_variants/$1
for f in ckkt.cu model_eval.cu mf_kernels.cuh dense_front.cuh analysis.h analysis.cpp; do git show $2:paper_2403_15913_b200/csrc/$f > $d/x/csrc/$f; done
git show $2:include/ckkt.h > $d/include/ckkt.h
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Xptxas -O3 \
  --expt-relaxed-constexpr $3 -c $d/x/csrc/ckkt.cu -o build_variants/$1/ckkt.o 2>&1 | grep -E "error" || true
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -c $d/x/csrc/model_eval.cu -o build_variants/$1/model_eval.o
g++ -O3 -fPIC -std=c++17 -c $d/x/csrc/analysis.cpp -I $d/include -o build_variants/$1/analysis.o
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o build_variants/$1/libckkt.so build_variants/$1/ckkt.o \
  build_variants/$1/model_eval.o build_variants/$1/analysis.o -lcudart
echo build_variants/$1/libckkt.so
