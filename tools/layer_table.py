"""Aggregate an ncu launch-list csv (gpu__time_duration.sum) per kernel name."""
import collections, csv, sys
rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
gi = h.index("Grid Size") if "Grid Size" in h else None
agg = collections.OrderedDict()
for x in rows[1:]:
    if len(x) != len(h) or x[mi] != "gpu__time_duration.sum":
        continue
    k = x[ki].split("(")[0].replace("(anonymous namespace)::", "").replace("hy::", "")
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += float(x[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"total {tot/1000:.1f} us, {sum(v[0] for v in agg.values())} launches")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:50]:50s} {n:6d} {t/1000:10.1f} us {100*t/tot:5.1f}%  avg {t/n/1000:8.1f}")
