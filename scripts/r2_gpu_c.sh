#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2c_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/r2c_gputest.log
timeout 600 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
bash scripts/r2_sanitize.sh
