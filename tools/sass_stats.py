"""Per-function SASS instruction histogram of the built library (CPU-side check)."""
import re, subprocess, sys, collections
lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1810_03358_b200/_lib/libffmin_b200.so"
pat = sys.argv[2] if len(sys.argv) > 2 else "nb_units_kernelIfLb1ELb0"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0]
    if pat not in name:
        continue
    ops = collections.Counter(re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", f))
    keys = ["FFMA2", "FMUL2", "FADD2", "FFMA", "FMUL", "FADD", "MUFU.RSQ", "SHFL.IDX", "LDS.128", "LDS.64", "MOV", "FSEL", "IMAD.MOV.U32"]
    print(name[:60], sum(ops.values()), {k: ops[k] for k in keys if ops[k]})
