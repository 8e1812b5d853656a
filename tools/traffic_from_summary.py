"""Rebuild profiles/ncu_traffic.json from a committed summary (profiles/<tag>_ncu_summary.md), e.g. after the
family mapping in tools/ncu_round.py changed:  python tools/traffic_from_summary.py <tag>"""
import collections
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_round as nr  # noqa: E402

tag = sys.argv[1]
md = open(os.path.join(nr.PROF, f"{tag}_ncu_summary.md")).read()
acc = collections.defaultdict(list)
for sec in re.split(r"^### ", md, flags=re.M)[1:]:
    kn = re.search(r"Kernel Name\s+(.*)", sec).group(1)
    rd = float(re.search(r"dram__bytes_read.sum\s+([\d.]+)", sec).group(1))
    wr = float(re.search(r"dram__bytes_write.sum\s+([\d.]+)", sec).group(1))
    fam, short = nr.family(kn)
    if fam:
        acc[fam].append((short, rd + wr))
t = {"source": f"profiles/{tag}_ncu_summary.md (ncu --set full, one launch per kernel)", "families": {}}
for fam, lst in acc.items():
    t["families"][fam] = {"kernel": " + ".join(k for k, _ in lst), "dram_bytes": sum(b for _, b in lst) / len(lst),
                          "items": int(os.environ.get("HY_ITEMS", "64"))}
json.dump(t, open(os.path.join(nr.PROF, "ncu_traffic.json"), "w"), indent=1)
print(json.dumps(t, indent=1))
