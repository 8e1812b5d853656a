#!/bin/bash
# quick GPU iteration: parity tests + short bench with per-family breakdown. $1 = tag
TAG=${1:-q}
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-conv > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -3 gpurun_out/bench_$TAG.err
python - << PY
import json; d=json.load(open("gpurun_out/bench_$TAG.json"))
print("value", round(d["value"],1), "ms", round(d["ms_per_step"],3), "hoisted", round(d["hoisted"]["value"],1), "launches", d["gpu_launches"])
for k,v in d["kernel_breakdown"].items(): print(f'  {k:8s} {v["ms_per_step"]:7.3f} ms/step {v["launches_per_step"]:5d} launches avg {v["avg_us"]:7.1f} us  {v["alg_bytes_per_launch"]/v["avg_us"]/1e3:7.1f} GB/s')
print("hoisted:")
for k,v in d["hoisted"].get("kernel_breakdown", {}).items(): print(f'  {k:8s} {v["ms_per_step"]:7.3f} ms/step {v["launches_per_step"]:5d} launches avg {v["avg_us"]:7.1f} us  {v["alg_bytes_per_launch"]/v["avg_us"]/1e3:7.1f} GB/s')
PY
