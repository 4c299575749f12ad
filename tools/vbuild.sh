#!/bin/bash
# build exp/<name>.so with extra flags (no GPU steps)
cd /root/repo
name=$1; shift
C=paper_1606_00519_b200/csrc
mkdir -p exp
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -Xptxas -v -I include -I $C "$@" -o exp/$name.so $C/*.cu $C/*.cpp -lpthread 2> exp/$name.ptxas
grep -A1 "huff_warp_kernelILb0ELj2" exp/$name.ptxas | grep -o "Used [0-9]* registers.*" | head -2
