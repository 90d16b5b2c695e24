#!/bin/bash
# build_variant.sh NAME UNIT "-DFLAGS ..." : libofdmr_b200_NAME.so with UNIT recompiled under FLAGS
set -e
cd "$(dirname "$0")/../paper_2209_03883_b200"
name=$1; unit=$2; shift 2
mkdir -p _build_v
nvcc -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a "$@" -c csrc/$unit.cu -o _build_v/${unit}_$name.o
objs=""
for o in _build/*.o; do b=$(basename $o .o); if [ "$b" = "$unit" ]; then objs="$objs _build_v/${unit}_$name.o"; else objs="$objs $o"; fi; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libofdmr_b200_$name.so $objs -lcudart
