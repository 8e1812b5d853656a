#!/bin/bash
# A/B of an env toggle on the HRot bench: $1 = tag, $2 = env assignment for the B arm (e.g. HY_FUSE_IP=0)
TAG=$1; ENVB=$2
for arm in A B; do
  if [ $arm = B ]; then export $ENVB; fi
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-conv --no-r18 > gpurun_out/ab_${TAG}_$arm.json 2>/dev/null
  python - << PY
import json; d=json.load(open("gpurun_out/ab_${TAG}_$arm.json"))
print("$arm", "value", round(d["value"],1), "ms", round(d["ms_per_step"],3), "hoisted", round(d["hoisted"]["value"],1))
for k,v in d["kernel_breakdown"].items(): print(f'  {k:8s} {v["ms_per_step"]:7.3f} ms/step {v["launches_per_step"]:5d} launches avg {v["avg_us"]:7.1f} us  {v["alg_bytes_per_launch"]/v["avg_us"]/1e3:7.1f} GB/s')
PY
done
