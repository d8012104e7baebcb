#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2h_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/r2h_gputest.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2h_bench.json 2>&1
timeout 1500 python bench_longtail.py --prompts 288 --max-inflight 384 --theta 32 --max-len 4096 \
  --late-join 256 --kv-gb 70 > gpurun_out/r2h_longtail.json 2> gpurun_out/r2h_longtail.err
timeout 1500 python bench_longtail.py > gpurun_out/r2h_longtail_default.json 2> gpurun_out/r2h_longtail_default.err
