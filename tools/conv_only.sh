#!/bin/bash
# conv-layer timings with per-family breakdown (no HRot micro, no CPU baseline): $1 = tag
python - "$1" << 'PY'
import json, subprocess, sys
tag = sys.argv[1]
out = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu-baseline"],
                     capture_output=True, text=True)
open(f"gpurun_out/conv_{tag}.json", "w").write(out.stdout)
d = json.loads(out.stdout.strip().splitlines()[-1])
print("hrot", round(d["value"], 1), "hoisted", round(d["hoisted"]["value"], 1))
for net in ("resnet20_conv", "resnet18_conv"):
    c = d[net]
    if not c: continue
    print(net, "total", round(c["total_ms"], 2))
    for k, v in c["layers"].items():
        print(f'  {k:10s} {v["ms"]:8.3f} ms x{v["mult"]}  ' + " ".join(f"{a}={b}" for a, b in v["family_ms"].items()))
PY
