#!/bin/bash
# build_variant.sh NAME "-DFLAG=..." : the native library with extra nvcc
# flags for tile.cu only, as build/var/NAME.so (experiments; PM_NATIVE_LIB)
set -e
cd "$(dirname "$0")/.."
mkdir -p build/var
objs=$(ls build/obj/*.o | grep -v tile.cu.o)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
  --expt-relaxed-constexpr -diag-suppress 128 -I include -I paper_1604_05937_b200/csrc $2 \
  -c paper_1604_05937_b200/csrc/tile.cu -o build/var/$1.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var/$1.so $objs build/var/$1.o
