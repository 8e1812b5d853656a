#!/bin/bash
# ncu --set full of one MulFilter&Sum launch of ResNet-18 L1_ca (PRCR) and L2_ds (no PRot) per kernel variant
# (HY_PMB_ROWS = 0 gather, 2 ring); summaries in gpurun_out/pmult_<layer>_<v>.txt.  $1 = tag
TAG=${1:-pm}
for L in L1_ca L2_ds; do
  for V in 0 2; do
    HY_PMB_ROWS=$V ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:k_pmult -s 2 -c 1 -o gpurun_out/${TAG}_${L}_$V python tools/prof_layer.py R18 $L --ncu > /dev/null 2>&1
    ncu -i gpurun_out/${TAG}_${L}_$V.ncu-rep --page raw --csv > gpurun_out/${TAG}_${L}_$V.csv 2>/dev/null
    python tools/ncu_sass_summary.py gpurun_out/${TAG}_${L}_$V.ncu-rep 12 > gpurun_out/${TAG}_${L}_${V}_sass.txt 2>&1
  done
done
