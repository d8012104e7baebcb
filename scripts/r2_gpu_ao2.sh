#!/bin/bash
# config 5 on the split-sum build: 2 GPUs, late joiner, theta 32 and 400
cd "$(dirname "$0")/.."
timeout 1500 python bench_longtail.py --instances 2 --prompts 192 --max-inflight 384 --theta 32 \
  --max-len 4096 --late-join 256 --kv-gb 70 > gpurun_out/r2ao_longtail2_t32.json 2> gpurun_out/r2ao_longtail2_t32.err
timeout 1500 python bench_longtail.py --instances 2 --prompts 192 --max-inflight 384 --theta 400 \
  --max-len 4096 --late-join 256 --kv-gb 70 > gpurun_out/r2ao_longtail2_t400.json 2> gpurun_out/r2ao_longtail2_t400.err
