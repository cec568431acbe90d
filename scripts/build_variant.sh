#!/bin/bash
# build_variant.sh NAME "-DFLAG=.. ..."  -> paper_2505_13723_b200/_lib_NAME/libsapgp_b200.so
# (the in-tree objects with the tensor-core kernels recompiled under the given flags)
set -e
name=$1; flags=$2
cd "$(dirname "$0")/../paper_2505_13723_b200/csrc"
d=../_lib_$name
mkdir -p $d/obj && cp ../_lib/obj/*.o $d/obj/
for f in krows_tc_m32 krows_tc_m52 krows_tc_rbf; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $flags -c $f.cu -o $d/obj/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libsapgp_b200.so $d/obj/*.o
