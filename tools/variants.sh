#!/bin/bash
# Build kernel variants of libphfem_b200.so side by side (in-tree, so they
# travel to the GPU box):  bash tools/variants.sh NAME "-DFLAG=.." [NAME "-D.."]...
# -> paper_2401_15557_b200/variants/libphfem_b200_NAME.so ; run one with
#    PHFEM_LIB=paper_2401_15557_b200/variants/libphfem_b200_NAME.so python bench.py ...
set -e
cd "$(dirname "$0")/../paper_2401_15557_b200/csrc"
mkdir -p ../variants
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  objs=()
  for f in $(sed -n 's/^SRCS *:= *//p' Makefile | sed 's/\.cu//g'); do
    nvcc -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
      -gencode arch=compute_100a,code=sm_100a $flags -c $f.cu -o /tmp/var_${name}_$f.o &
    objs+=(/tmp/var_${name}_$f.o)
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../variants/libphfem_b200_$name.so "${objs[@]}" -cudart static
  echo "built variants/libphfem_b200_$name.so"
done
