#!/bin/bash
# time every variant in _lib/variants twice, interleaved: tools/sweep_variants.sh [natoms] [prec] [grad]
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for lib in paper_1810_03358_b200/_lib/variants/lib_*.so; do
    v=$(basename $lib .so)
    echo "$v $(FFMIN_B200_LIB=$lib timeout 120 python tools/time_nb.py ${1:-100000} ${2:-1} ${3:-1} 2>&1 | tail -1)"
  done
done
