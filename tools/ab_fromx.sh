for r in 1 2 3; do
 for cfg in "0 0" "1500 0" "1500 1"; do set -- $cfg
  for p in f32 f64; do
   echo "maxn=$1 f64all=$2 $p $(FFM_SMALL_FROMX_MAXN=$1 FFM_SMALL_FROMX_F64=$2 PREC=$p VARIANTS=auto python tools/mid_sweep.py 500 1000 1500 | grep -o 'n= *[0-9]*\|eval= *[0-9.]*' | tr -s ' ' | tr '\n' ' ')"
  done
 done
done
