#!/bin/bash
# A/B of small-system evaluation time for every library in _lib/variants
# (tuning aid): whole-evaluation graph replay (mid_sweep) for FP32 / FP64 at
# 500-4000 atoms, plus the fused kernel's phase stamps at 3000 atoms FP32.
cd "$(dirname "$0")/.."
for r in 1 2; do
for L in paper_1810_03358_b200/_lib/variants/lib_*.so; do
  v=$(basename $L .so | sed 's/^lib_//')
  FFMIN_B200_LIB=$L VARIANTS=auto timeout 300 python tools/mid_sweep.py ${SIZES:-500 1000 2000 3000 4000} 2>&1 | grep "^n=" | sed "s/^/$v f32 /"
  FFMIN_B200_LIB=$L PREC=f64 VARIANTS=auto timeout 300 python tools/mid_sweep.py ${SIZES:-500 1000 2000 3000 4000} 2>&1 | grep "^n=" | sed "s/^/$v f64 /"
  [ $r = 1 ] && FFMIN_B200_LIB=$L timeout 100 python tools/time_small_phases.py 3000 1 1 2>&1 | sed "s/^/$v /"
done; done
