#!/bin/bash
# run tools/mid_sweep.py against every library in _lib/variants (tuning aid)
cd "$(dirname "$0")/.."
for lib in paper_1810_03358_b200/_lib/variants/lib_*.so; do
  v=$(basename $lib .so)
  FFMIN_B200_LIB=$lib timeout 300 python tools/mid_sweep.py "$@" 2>&1 | grep "^n=" | sed "s/^/$v /"
done
