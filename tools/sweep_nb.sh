#!/bin/bash
cd "$(dirname "$0")/.."
for lib in paper_1810_03358_b200/_lib/variants/lib_*.so; do
  v=$(basename $lib .so)
  echo "$v f32grad $(FFMIN_B200_LIB=$lib python tools/time_nb.py ${1:-100000} 1 1 2>/dev/null)"
  [ -n "$F64" ] && echo "$v f64grad $(FFMIN_B200_LIB=$lib python tools/time_nb.py ${1:-100000} 0 1 2>/dev/null)"
done
