#!/bin/bash
# split-K sweep for the decode-step projections (1.5B shape), warm re-launch timings
for s in "4,6,5" "2,2,5" "4,4,4" "2,3,4" "4,4,7"; do
  echo "splits=$s"
  RLB_SPLITS=$s timeout 300 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --prompts 512 --new-tokens 1024 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); k=d['kernels_mid_rollout']
print(round(d['value']), {n: k[n]['avg_ms']*1000 for n in ('qkv','o_proj','down')})"
done
