#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python bench_migrate.py --check > gpurun_out/r2y_migrate4.json 2> gpurun_out/r2y_migrate4.err
CUDA_VISIBLE_DEVICES=0 timeout 900 python scripts/decode_profile.py gpurun_out/r2y_decode_profile.json > gpurun_out/r2y_decode_profile.log 2>&1
CUDA_VISIBLE_DEVICES=1 timeout 900 python scripts/decode_profile.py gpurun_out/r2y_decode_profile_7b.json --shape qwen2.5-7b > gpurun_out/r2y_decode_profile_7b.log 2>&1
