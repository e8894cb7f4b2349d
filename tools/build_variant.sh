#!/bin/bash
# build/libgbbs_<name>.so with extra -D flags (dev tool for A/B runs via GBBS_LIB)
name=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared --expt-relaxed-constexpr "$@" -Xptxas -v \
  -o build/libgbbs_$name.so paper_1805_05208_b200/csrc/gbbs.cu 2> build/$name.ptxas.log
grep -A1 "traverse_kernelILi1ELb0" build/$name.ptxas.log | grep -E "spill|Used" | head -2
