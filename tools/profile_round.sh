#!/bin/bash
# Round evidence: launch list of the bench's timed regions + ncu --set full of every distinct kernel in it.
# usage: tools/profile_round.sh <tag>   (run from the repo root under gpurun; then tools/ncu_round.py <tag>)
TAG=${1:-r01}
export HY_NCU_TIMED=1
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-conv --no-variants --no-c1"
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --kernel-name-base demangled --log-file gpurun_out/launches_${TAG}.csv $B > /dev/null 2>&1
# one full capture per distinct kernel (first launch in the timed region, which is the plain step's chunk 0
# for the kernels both steps share; the hoisted-only instantiations are captured from the hoisted step)
python - "$TAG" > gpurun_out/kernels_${TAG}.txt << 'PY'
import csv, re, sys
tag = sys.argv[1]
rows = list(csv.reader(l for l in open(f"gpurun_out/launches_{tag}.csv") if not l.startswith("==")))
h = rows[0]; ki = h.index("Kernel Name")
names = []
for x in rows[1:]:
    if len(x) != len(h) or x[h.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    names.append(x[ki].replace("(anonymous namespace)::", "").split("(")[0].replace("void ", "").strip().split("::")[-1])
seen = []
for n in names:
    if n not in seen:
        seen.append(n)
for n in seen:  # ncu -k regex:<base>[<(] counts only matching launches for --launch-skip
    base = n.split("<")[0]
    same = [m for m in names if m.split("<")[0] == base]
    print(base, same.index(n))
PY
i=0
while read -r k skip; do
  i=$((i+1))
  ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:${k}[<(]" -s $skip -c 1 -o gpurun_out/prof_${TAG}_k$i $B > /dev/null 2>&1
done < gpurun_out/kernels_${TAG}.txt
ls gpurun_out | grep $TAG
