#!/bin/bash
# A/B of an env switch on the C2 microbenchmark: tools/ab_env.sh VAR "v1 v2 ..." [pytest -k expr]
VAR=$1; VALS=$2; K=$3
if [ -n "$K" ]; then python -m pytest tests/test_gpu_parity.py -x -q -k "$K" 2>&1 | tail -3; fi
for v in $VALS; do
  env $VAR=$v python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-conv > gpurun_out/ab_${VAR}_$v.json 2> gpurun_out/ab_${VAR}_$v.err
  python - "$VAR" "$v" << 'PY'
import json, sys
var, v = sys.argv[1], sys.argv[2]
d = json.load(open(f"gpurun_out/ab_{var}_{v}.json"))
print(f"{var}={v}: plain {d['value']:.1f}/s  hoisted {d['hoisted']['value']:.1f}/s")
for tag, br in (("plain", d["kernel_breakdown"]), ("hoisted", d["hoisted"].get("kernel_breakdown", {}))):
    for k, x in br.items():
        print(f"   {tag:8s} {k:8s} {x['ms_per_step']:7.3f} ms/step {x['launches_per_step']:4d} launches {x['alg_bytes_per_launch']/x['avg_us']/1e3:7.1f} GB/s")
PY
done
