#!/bin/bash
# Build abtest/lib_NAME.so: the in-tree objects with csrc/FILE.cu recompiled
# from SRC (default: the in-tree source) with extra nvcc flags.
# usage: tools/variant.sh NAME FILE [SRC] [-DFLAG ...]
name=$1; file=$2; shift 2
src=paper_1602_00001_b200/csrc/$file.cu
if [ -n "$1" ] && [ "${1#-}" = "$1" ]; then src=$1; shift; fi
mkdir -p abtest build/variant
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
  --expt-relaxed-constexpr -I include -I paper_1602_00001_b200/csrc "$@" -c $src -o build/variant/$file.$name.o || exit 1
objs=$(ls build/csrc/*.o | grep -v "/$file.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o abtest/lib_$name.so $objs build/variant/$file.$name.o -lcudart
