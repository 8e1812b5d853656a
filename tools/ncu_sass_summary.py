"""Summarise an ncu report's SASS page: executed instructions per opcode and top stall lines."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hi = next(i for i, x in enumerate(r) if x and x[0] == "Address")
h = r[hi]
ii, si = h.index("Instructions Executed"), h.index("Source")
wi = h.index("Warp Stall Sampling (All Samples)")
rows = [x for x in r[hi + 1:] if len(x) == len(h)]
op = collections.Counter()
stall = collections.Counter()
tot = 0
for x in rows:
    n = int(x[ii] or 0)
    tot += n
    o = x[si].strip().split()[0] if x[si].strip() else "?"
    if o.startswith("@"):
        o = x[si].strip().split()[1]
    o = o.split(".")[0]
    op[o] += n
    stall[o] += int(x[wi] or 0)
print(f"total warp-instructions executed: {tot}")
for o, n in op.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 15):
    print(f"  {o:12s} {n:12d} {100*n/tot:5.1f}%  stall-samples {stall[o]}")
