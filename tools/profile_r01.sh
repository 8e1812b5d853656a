#!/bin/bash
# ncu evidence for the bench's timed region (run under gpurun from the repo root).
# $1 = tag (e.g. r01a)
set -x
TAG=${1:-r01}
export HY_NCU_TIMED=1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for k in k_ntt_rows k_ntt_cols256 k_modup_bconv k_ks_ip k_moddown_bconv k_moddown_final k_automorph; do
  ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$k -c 1 \
      -o gpurun_out/prof_${TAG}_$k python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
ls -la gpurun_out/
