#!/bin/bash
# bench.py under several tuning environments: "ENV=.. ENV2=.." per argument.
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | python scripts/bench_summary.py "$cfg"
done
