#!/bin/bash
# Dev helper: build a timing variant of the library with extra nvcc flags into exp/<name>.so
# (tools/lzexp_time.py times libgompresso.so beside every exp/*.so). Usage: variant_build.sh name -DFOO=1 ...
cd "$(dirname "$0")/.."
name=$1; shift
C=paper_1606_00519_b200/csrc
mkdir -p exp
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -I include -I $C "$@" -o exp/$name.so $C/*.cu $C/*.cpp -lpthread
