#!/bin/bash
# full GPU suite on the split-sum build + prefill chunk size A/B (16384 vs 18944 = 74 x 256)
cd "$(dirname "$0")/.."
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2ad_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/r2ad_gputest.log
for r in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline --steps 2 --prefill-rows 18944 > gpurun_out/r2ad_bench_18944_$r.json 2>&1
  timeout 600 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/r2ad_bench_16384_$r.json 2>&1
done
