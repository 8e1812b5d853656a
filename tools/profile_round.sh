#!/bin/bash
# Round evidence: launch list of the bench's timed regions + ncu --set full of the hot kernels.
# usage: tools/profile_round.sh <tag>   (run from the repo root under gpurun; then tools/ncu_round.py <tag>)
TAG=${1:-r01}
export HY_NCU_TIMED=1
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-conv"
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv $B > /dev/null 2>&1
i=0
# demangled names print bool template arguments as 0 / 1
for k in "k_bconv_cols<4, 0>" "k_bconv_cols<4, 1>" "k_rows_ip_final_tma<6, 0, 2>" "k_rows_ip_final_tma<6, 1, 2>" \
         "k_ntt_rows_ip<6, 0>" "k_ntt_rows<0>" "k_automorph" "k_ks_ip<6, 0, 0>" "k_modup_bconv<4>"; do
  i=$((i+1))
  ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"${k}" -s 2 -c 1 \
      -o gpurun_out/prof_${TAG}_k$i $B > /dev/null 2>&1
done
ls gpurun_out | grep $TAG
