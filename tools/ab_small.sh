for r in 1 2; do
for v in old new; do
  L=paper_1810_03358_b200/_lib/variants/lib_$v.so
  FFMIN_B200_LIB=$L VARIANTS=auto timeout 300 python tools/mid_sweep.py 500 1000 2000 3000 4000 2>&1 | grep "^n=" | sed "s/^/$v f32 /"
  FFMIN_B200_LIB=$L PREC=f64 VARIANTS=auto timeout 300 python tools/mid_sweep.py 500 1000 2000 3000 4000 2>&1 | grep "^n=" | sed "s/^/$v f64 /"
  FFMIN_B200_LIB=$L timeout 100 python tools/time_small_phases.py 3000 0 1 2>&1 | sed "s/^/$v /"
done; done
