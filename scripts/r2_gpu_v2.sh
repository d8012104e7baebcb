#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1500 python bench_longtail.py --instances 2 --prompts 192 --max-inflight 384 --theta 400 \
  --max-len 4096 --late-join 256 --kv-gb 70 > gpurun_out/r2v_longtail2.json 2> gpurun_out/r2v_longtail2.err
timeout 900 python scripts/kernel_dbg.py > gpurun_out/r2v_kernel_dbg.txt 2>&1
