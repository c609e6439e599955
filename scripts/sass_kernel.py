"""Static SASS view of one kernel of libbsgpu.so: python scripts/sass_kernel.py <substring of the
mangled name> [lo hi] — lists the instructions between addresses lo and hi (hex), or, without a range,
the instruction count between consecutive mbarrier try-waits (one per plane or plane pair of a sweep)."""
import re
import subprocess
import sys
from collections import Counter

lib = "paper_2009_12638_b200/_lib/libbsgpu.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
name = sys.argv[1]
ins = []
on = False
for line in out.split("\n"):
    if "Function :" in line:
        on = name in line
        continue
    if on:
        m = re.match(r"\s+/\*([0-9a-f]{4,6})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
print(len(ins), "instructions")
if len(sys.argv) >= 4:
    lo, hi = int(sys.argv[2], 16), int(sys.argv[3], 16)
    sel = [(a, t) for a, t in ins if lo <= a <= hi]
    for a, t in sel:
        print(f"{a:05x} {t}")
    c = Counter((t.split()[1] if t.startswith("@") else t.split()[0]) for _, t in sel)
    print(len(sel), dict(c.most_common(20)))
else:
    waits = [i for i, (_, t) in enumerate(ins) if "TRYWAIT" in t]
    prev = None
    for i in waits:
        if prev is not None:
            seg = ins[prev:i]
            c = Counter((t.split()[1] if t.startswith("@") else t.split()[0]) for _, t in seg)
            dp = sum(v for k, v in c.items() if k.startswith(("DADD", "DMUL", "DFMA")))
            print(f"{ins[prev][0]:05x}-{ins[i][0]:05x} n={len(seg)} dp={dp} lds={c.get('LDS.64', 0)} bra={c.get('BRA', 0)}")
        prev = i
