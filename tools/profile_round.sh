#!/bin/bash
# Round evidence: launch list of the bench's timed regions + ncu --set full of the hot kernels.
# usage: tools/profile_round.sh <tag>   (run from the repo root under gpurun; then tools/ncu_round.py <tag>)
TAG=${1:-r01}
export HY_NCU_TIMED=1
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-conv"
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv $B > /dev/null 2>&1
for k in k_modup_cols k_rows_ip_final k_ntt_rows_ip k_ntt_rows_final k_moddown_bconv k_ntt_cols256 k_ntt_rows k_automorph \
         k_ks_ip k_modup_bconv; do
  ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"${k}[<(]" -s 2 -c 1 \
      -o gpurun_out/prof_${TAG}_$k $B > /dev/null 2>&1
done
ls gpurun_out | grep $TAG
