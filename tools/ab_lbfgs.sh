#!/bin/bash
# graph-resident FP64 L-BFGS per iteration for every library in _lib/variants (tuning aid)
cd "$(dirname "$0")/.."
for r in 1 2; do
for L in paper_1810_03358_b200/_lib/variants/lib_*.so; do
  v=$(basename $L .so | sed 's/^lib_//')
  for n in ${SIZES:-20 500 1000 2000}; do
    echo "$v $(FFMIN_B200_LIB=$L timeout 120 python tools/lbfgs_launches.py $n 0 300)"
  done
done; done
