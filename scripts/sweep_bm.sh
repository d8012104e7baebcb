#!/bin/bash
# Tile-height (RLB_BM = qkv,o,gate_up,down rows per CTA; tile shapes never
# change a row's bits) x O/down split-K sweep of the decode-step projections
# (1.5B shape): tokens/s, decode ms/step, warm kernels.
#   scripts/sweep_bm.sh 128,128,256,256:3,5 ...
run() {
  echo "BM=$1 SPLITS(o,down)=$2"
  env RLB_BM=$1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
    --split-o ${2%,*} --split-down ${2#*,} 2>/dev/null | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); k=d['kernels_mid_rollout']; ph=d['phases_ms_rank0']
print(' ', round(d['value']), 'decode ms/step', round(ph['decode']/ph['decode_steps'],3), 'prefill ms', ph['prefill'],
      {n: round(k[n]['avg_ms']*1000,1) for n in k})"
}
for cfg in "$@"; do
  run ${cfg//:/ }
done
