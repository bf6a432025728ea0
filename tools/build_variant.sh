#!/bin/bash
# build_variant.sh NAME "-DFLAG=..." [SRC] : the native library with extra
# nvcc flags for one source file (default tile.cu) as build/var/NAME.so
# (experiments; load with PM_NATIVE_LIB=build/var/NAME.so)
set -e
cd "$(dirname "$0")/.."
src=${3:-tile.cu}
mkdir -p build/var
objs=$(ls build/obj/*.o | grep -v "/$src.o")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
  --expt-relaxed-constexpr -diag-suppress 128 -I include -I paper_1604_05937_b200/csrc $2 \
  -c paper_1604_05937_b200/csrc/$src -o build/var/$1.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var/$1.so $objs build/var/$1.o
