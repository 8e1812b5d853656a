"""Per-source-line stall samples (with the top stall reasons) from
`ncu -i X --page source --csv --print-source cuda,sass` output.  usage: python tools/src_stalls.py file.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, lines, hdr = "?", [], None
for r in rows:
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0] not in ("",) and r[0].isdigit() and len(r) == len(hdr):
        lines.append((fname, r))
iN = hdr.index("Warp Stall Sampling (All Samples)")
iX = hdr.index("Instructions Executed")
stall_cols = [i for i, x in enumerate(hdr) if x.startswith("stall_")]
tot = sum(int(r[iN]) for _, r in lines if r[iN].isdigit())
print("total samples", tot)
for f, r in sorted(lines, key=lambda t: -int(t[1][iN]) if t[1][iN].isdigit() else 0)[:top]:
    n = int(r[iN])
    st = sorted(((int(r[i]) if r[i].isdigit() else 0, hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
    print(f"{100 * n / tot:5.1f}% {f}:{r[0]:5s} x={r[iX]:>10s} [{' '.join(f'{k}:{100*v/max(n,1):.0f}' for v, k in st)}] {r[1].strip()[:90]}")
