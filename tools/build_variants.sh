#!/bin/bash
# Tuning sweep: rebuild the pair kernel with different unroll / schedule
# choices into _lib/variants/ (development aid, results in profiles/).
set -e
cd "$(dirname "$0")/.."
L=paper_1810_03358_b200/_lib
mkdir -p $L/variants $L/obj
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC"
for src in ffm_terms ffm_vec ffm_capi; do
  extra=""; [ $src = ffm_terms ] && extra="-fmad=false"
  nvcc $F $extra -c -o $L/obj/$src.o paper_1810_03358_b200/csrc/$src.cu &
done
wait
for v in "$@"; do
  u=${v%_*}; s=${v#*_}
  (nvcc $F -DFFM_UNROLL=$u -DFFM_SCHED=$s -DFFM_MINB=${MINB:-2} -DFFM_PAIRFMA=${PAIRFMA:-0} -DFFM_VFMA=${VFMA:-1} -c -o $L/obj/pairs_${v}_vf${VFMA:-1}.o paper_1810_03358_b200/csrc/ffm_pairs.cu -Xptxas -v 2>&1 | grep -A1 "nb_units_kernelIfLb1ELb0" | grep -oE "Used [0-9]+ registers|[0-9]+ bytes spill stores" | tr '\n' ' '; echo " <- $v"
   nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $L/variants/lib_${v}_vf${VFMA:-1}.so $L/obj/pairs_${v}_vf${VFMA:-1}.o $L/obj/ffm_terms.o $L/obj/ffm_vec.o $L/obj/ffm_capi.o) &
done
wait
