"""Instruction mix (ALU vs FMA pipe) of one kernel's SASS, for comparing
field-arithmetic variants on the CPU before spending GPU time.
usage: python tools/sass_mix.py <object or .so> <kernel-name regex>"""
import re
import subprocess
import sys
from collections import Counter

ALU = ("IADD3", "LOP3", "SEL", "SHF", "LEA", "ISETP", "PRMT", "VIADD", "IMNMX", "FSEL", "PLOP3", "MOV")
FMA = ("IMAD", "FFMA", "HFMA2")

obj, pat = sys.argv[1], re.compile(sys.argv[2])
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", sass)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if not pat.search(name):
        continue
    ops = Counter()
    for m in re.finditer(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", f):
        ops[m.group(1)] += 1
    alu = sum(v for k, v in ops.items() if k.split(".")[0] in ALU)
    fma = sum(v for k, v in ops.items() if k.split(".")[0] in FMA)
    print(f"{name[:110]}\n  total {sum(ops.values())}  alu {alu}  fma {fma}  top {ops.most_common(8)}")
