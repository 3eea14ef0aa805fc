#!/bin/bash
# Build libdmas variants that differ only in dmas_envelope_tc.cu macros (experiments):
#   tools/build_variants.sh NAME "-DMACRO=V ..." [NAME2 "..."]...  -> paper_2511_09165_b200/build/libdmas_NAME.so
set -e
cd "$(dirname "$0")/.."
B=paper_2511_09165_b200/build
FLAGS="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC,-ffp-contract=off,-O2 -I include -I paper_2511_09165_b200/csrc"
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  nvcc $FLAGS $defs -c -o $B/env_$name.o paper_2511_09165_b200/csrc/dmas_envelope_tc.cu &
done
wait
for o in $B/env_*.o; do
  name=$(basename $o .o); name=${name#env_}
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $B/libdmas_$name.so $B/dmas_kernels.cu.o $o $B/dmas_plan.cpp.o $B/dmas_comm.cpp.o -ldl
  echo $B/libdmas_$name.so
done
