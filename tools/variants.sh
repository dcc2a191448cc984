#!/bin/bash
# Build pair-kernel variants: tools/variants.sh NAME "-DFLAG=.. -DFLAG2=.." [NAME2 "FLAGS2" ...]
# -> paper_1810_03358_b200/_lib/variants/lib_NAME.so (time with FFMIN_B200_LIB=... tools/time_nb.py)
set -e
cd "$(dirname "$0")/.."
L=paper_1810_03358_b200/_lib
C=paper_1810_03358_b200/csrc
mkdir -p $L/variants $L/obj
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC"
for src in ffm_terms ffm_small ffm_vec ffm_minimize ffm_capi; do
  extra=""; { [ $src = ffm_terms ] || [ $src = ffm_small ] || [ $src = ffm_minimize ]; } && extra="-fmad=false"
  nvcc $F $extra -c -o $L/obj/$src.o $C/$src.cu &
done
wait
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  (nvcc $F $flags -c -o $L/obj/pairs_$name.o $C/ffm_pairs.cu -Xptxas -v 2>&1 \
     | grep -A2 "Compiling entry function '_ZN3ffm15nb_units_kernelIfLb1ELb0" \
     | grep -oE "Used [0-9]+ registers|[0-9]+ bytes spill stores" | tr '\n' ' '; echo " <- $name ($flags)"
   nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $L/variants/lib_$name.so \
     $L/obj/pairs_$name.o $L/obj/ffm_terms.o $L/obj/ffm_small.o $L/obj/ffm_vec.o $L/obj/ffm_minimize.o $L/obj/ffm_capi.o) &
done
wait
