#!/bin/bash
# full ncu capture of selected kernels from the bench timed region. $1 = tag, rest = kernel regexes
TAG=$1; shift
export HY_NCU_TIMED=1
for k in "$@"; do
  ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
      -o gpurun_out/prof_${TAG}_$k python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
ls gpurun_out/ | grep $TAG
