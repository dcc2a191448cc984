"""Table of tools/ab_small.sh output: evaluation us per (precision, N, variant)."""
import collections
import sys

ev = collections.defaultdict(list)
for line in open(sys.argv[1]):
    f = line.split()
    if len(f) > 14 and f[2] == "n=":
        ev[(f[1], int(f[3]), f[0])].append(float(f[13]))
vs = sorted({k[2] for k in ev})
for prec in ("f32", "f64"):
    print(prec, "N".rjust(6), *[v.rjust(8) for v in vs])
    for n in sorted({k[1] for k in ev if k[0] == prec}):
        print("   ", str(n).rjust(6), *[f"{min(ev[(prec, n, v)]):8.1f}" if ev[(prec, n, v)] else " " * 8 for v in vs])
