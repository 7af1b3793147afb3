#!/bin/bash
# Development aid: build a variant of the library (extra nvcc flags) into scratch_libs/lib_<name>.so
# usage: scripts/build_variant.sh <name> "<extra flags>"
set -e
cd "$(dirname "$0")/../paper_1810_01967_b200/csrc"
NAME=$1; EXTRA=$2
B=build_$NAME
mkdir -p $B ../../scratch_libs
NV="/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Xptxas -v $EXTRA"
# only cbb_project.cu differs between variants; the other objects come from the main build
$NV -c cbb_project.cu -o $B/cbb_project.o 2> $B/cbb_project.ptxas.log || (cat $B/cbb_project.ptxas.log; false)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../scratch_libs/lib_$NAME.so \
  build/cbb_capi.o $B/cbb_project.o build/cbb_operator.o build/cbb_graph.o -L/usr/local/cuda/lib64 -lcufft \
  -Xlinker -rpath=/usr/local/cuda/lib64 -Xcompiler -fvisibility=hidden
echo built scratch_libs/lib_$NAME.so
