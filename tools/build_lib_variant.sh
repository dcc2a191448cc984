#!/bin/bash
# Build a complete engine library with extra -D flags into _lib/variants/lib_NAME.so
# (tuning aid): tools/build_lib_variant.sh NAME "-DFOO=1 -DBAR=2"
set -e
cd "$(dirname "$0")/.."
L=paper_1810_03358_b200/_lib
mkdir -p $L/variants $L/obj_$1
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $2"
objs=""
for src in ffm_pairs ffm_terms ffm_small ffm_vec ffm_minimize ffm_capi; do
  extra=""; case $src in ffm_terms|ffm_small|ffm_minimize) extra="-fmad=false";; esac
  nvcc $F $extra -c -o $L/obj_$1/$src.o paper_1810_03358_b200/csrc/$src.cu &
  objs="$objs $L/obj_$1/$src.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $L/variants/lib_$1.so $objs
rm -rf $L/obj_$1
