#!/bin/bash
# Builds libvcgpu.so with extra -D flags into variants/NAME/ (A/B runs, outside the package:
# VCGPU_LIB=variants/NAME/libvcgpu.so python tools/probe.py c5).
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
OUT=variants/$NAME
mkdir -p $OUT/obj
SRC=paper_2204_10402_b200/csrc
for f in $SRC/*.cu; do
  b=$(basename $f .cu)
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xptxas -v -Xcompiler -fPIC,-fvisibility=hidden "$@" -c $f -o $OUT/obj/$b.cu.o 2> $OUT/obj/$b.ptxas.log &
done
for f in $SRC/*.cpp; do
  b=$(basename $f .cpp)
  g++ -O3 -std=c++17 -fPIC -fvisibility=hidden "$@" -c $f -o $OUT/obj/$b.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libvcgpu.so $OUT/obj/*.o -Xlinker --exclude-libs,ALL -Xlinker -Bsymbolic
grep -A2 "dense_kernelILi16ELb0" $OUT/obj/dense_engine.ptxas.log | tail -2
