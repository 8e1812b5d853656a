#!/bin/bash
# sweep the key-switch batch cap and the NTT chunk size on the HRot bench
for B in 1 2 4 16; do for C in 64 256; do
  HY_KS_BATCH=$B HY_NTT_CHUNK=$C python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-conv > /tmp/b.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/b.json')); print('batch $B chunk $C', round(d['value'],1), 'hoisted', round(d['hoisted']['value'],1), {k: round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()})"
done; done
for B in 1 4 16; do
  HY_KS_BATCH=$B HY_NTT_CHUNK=64 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /tmp/c.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/c.json')); print('conv batch $B', round(d['resnet20_conv']['total_ms'],2), round(d['resnet18_conv']['total_ms'],2))"
done
