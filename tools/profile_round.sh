#!/bin/bash
# Round evidence: launch list of the bench's timed regions + ncu --set full of the hot kernels.
# usage: tools/profile_round.sh <tag>   (run from the repo root under gpurun; then tools/ncu_round.py <tag>)
TAG=${1:-r01}
export HY_NCU_TIMED=1
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-conv"
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv $B > /dev/null 2>&1
# (kernel regex, launches to skip) in the timed region's launch order: per 16-item chunk of the plain step
# k_bconv_cols runs ModUp (<4, 0>) then ModDown (<4, 1>); the plain Q-limb kernels (<6, 0, 2>) precede the
# hoisted ones (<6, 1, 2>) of the second timed step
i=0
for ks in "k_bconv_cols:2" "k_bconv_cols:3" "k_rows_ip_final_tma:2" "k_rows_ip_final_tma:5" "k_ntt_rows_ip:2" \
          "k_ntt_rows:2" "k_automorph:2" "k_ks_ip:1" "k_modup_bconv:0"; do
  i=$((i+1))
  k=${ks%%:*}; skip=${ks##*:}
  ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"${k}[<(]" -s $skip -c 1 \
      -o gpurun_out/prof_${TAG}_k$i $B > /dev/null 2>&1
done
ls gpurun_out | grep $TAG
