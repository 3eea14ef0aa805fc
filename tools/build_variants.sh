#!/bin/bash
# Build libdmas variants that differ only in the macros of ONE translation unit (experiments):
#   tools/build_variants.sh [-t kernels|env] NAME "-DMACRO=V ..." [NAME2 "..."]...
#     -> paper_2511_09165_b200/build/libdmas_NAME.so (the other objects from the last regular build)
set -e
cd "$(dirname "$0")/.."
B=paper_2511_09165_b200/build
TU=env
if [ "$1" = "-t" ]; then TU=$2; shift 2; fi
if [ "$TU" = "env" ]; then SRC=paper_2511_09165_b200/csrc/dmas_envelope_tc.cu; else SRC=paper_2511_09165_b200/csrc/dmas_kernels.cu; fi
FLAGS="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC,-ffp-contract=off,-O2 -I include -I paper_2511_09165_b200/csrc"
names=()
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  names+=($name)
  nvcc $FLAGS $defs -c -o $B/var_$name.o $SRC &
done
wait
for name in "${names[@]}"; do
  if [ "$TU" = "env" ]; then objs="$B/dmas_kernels.cu.o $B/var_$name.o"; else objs="$B/var_$name.o $B/dmas_envelope_tc.cu.o"; fi
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $B/libdmas_$name.so $objs $B/dmas_plan.cpp.o $B/dmas_comm.cpp.o -ldl
  echo $B/libdmas_$name.so
done
