#!/bin/bash
# Round evidence on the GPU box, sized for gpurun's 64 MiB copy-back: full bench line, launch list,
# ncu --set full of every timed kernel summarised there (tools/ncu_round.py), then the .ncu-rep removed.
# usage (under gpurun): bash tools/gpu_profile_round.sh <tag>
TAG=${1:-r01}
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
tail -2 gpurun_out/bench_${TAG}.err
timeout 1500 bash tools/profile_round.sh $TAG > /dev/null
python tools/ncu_round.py $TAG > /dev/null
mkdir -p gpurun_out/profiles
cp profiles/${TAG}_ncu_summary.md profiles/${TAG}_launches.csv profiles/ncu_traffic.json gpurun_out/profiles/
for f in gpurun_out/prof_${TAG}_*.ncu-rep; do
  ncu -i $f --page details --csv > ${f%.ncu-rep}_details.csv 2>/dev/null
  rm -f $f
done
du -sh gpurun_out
