#!/bin/bash
cd "$(dirname "$0")/.."
for pr in 16384 24576 32768; do
  timeout 600 python bench.py --no-cpu-baseline --steps 2 --prefill-rows $pr > gpurun_out/r2x_bench_pr$pr.json 2>&1
done
