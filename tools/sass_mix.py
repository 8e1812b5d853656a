"""Instruction mix and stall samples per opcode from an `ncu --page source --csv --print-source sass` export.
usage: python tools/sass_mix.py file.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
h = rows[1]
iS, iX, iN = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
ops = defaultdict(lambda: [0, 0])
tot_i = tot_s = 0
for r in rows[2:]:
    if len(r) < len(h) or not r[iX].isdigit():
        continue
    src = r[iS].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    x, n = int(r[iX] or 0), int(r[iN] or 0)
    ops[op][0] += x
    ops[op][1] += n
    tot_i += x
    tot_s += n
print(f"total warp instructions {tot_i:.3e}, stall samples {tot_s}")
for op, (x, n) in sorted(ops.items(), key=lambda t: -t[1][0])[:top]:
    print(f"{op:24s} {x:12d} {100 * x / tot_i:6.2f}%   samples {100 * n / max(tot_s, 1):6.2f}%")
