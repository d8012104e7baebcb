#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_engine.py -m gpu -q -p no:cacheprovider -k "split_sum" > gpurun_out/r2aq_test.log 2>&1
echo "rc=$?" >> gpurun_out/r2aq_test.log
