#!/bin/bash
# build an experiment variant of the library: scripts/build_variant.sh NAME -DMACRO=V ...
cd "$(dirname "$0")/../paper_1411_2239_b200/csrc"
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared "$@" \
  -o ../libltl4c_${name}.so compiler.cpp encoder.cpp partition.cu hot.cu seg.cu ingest.cu kernels.cu runtime.cu
