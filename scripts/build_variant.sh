#!/bin/bash
# build/var_<name>/libmrep.so: one source (SRC, default mrep_project) recompiled
# with extra nvcc flags, linked with the other objects of the current build
# (A/B runs with MREP_LIB=build/var_<name>/libmrep.so)
set -e
name=$1; shift
cd "$(dirname "$0")/.."
mkdir -p build/var_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -ffp-contract=off -Xcompiler -fvisibility=hidden -I include "$@" \
  -c paper_2504_11498_b200/csrc/${SRC:-mrep_project}.cu -o build/var_$name/${SRC:-mrep_project}.o
objs=$(ls build/*.o | grep -v ${SRC:-mrep_project}.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var_$name/libmrep.so build/var_$name/${SRC:-mrep_project}.o $objs -lcudart_static -lrt -lpthread -ldl
