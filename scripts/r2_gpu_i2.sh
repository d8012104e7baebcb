#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1500 python bench_longtail.py --instances 2 --prompts 192 --max-inflight 384 --theta 32 \
  --max-len 4096 --late-join 256 --kv-gb 70 > gpurun_out/r2i_longtail2.json 2> gpurun_out/r2i_longtail2.err
for pr in 2048 4096 8192 16384; do
  CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-cpu-baseline --steps 1 --prefill-rows $pr \
    > gpurun_out/r2i_bench_pr$pr.json 2>&1
done
