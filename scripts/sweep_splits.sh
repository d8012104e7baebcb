#!/bin/bash
# split-K sweep of the O / down projections (1.5B shape; part of the numerics
# plan, so each point is a different plan): tokens/s and warm kernel timings
for s in "3,5" "2,5" "4,4" "3,4" "4,7"; do
  o=${s%,*}; d=${s#*,}
  echo "split_o=$o split_down=$d"
  timeout 300 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --split-o $o --split-down $d \
    2>/dev/null | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); k=d['kernels_mid_rollout']
print(round(d['value']), {n: k[n]['avg_ms']*1000 for n in ('qkv','o_proj','down')})"
done
