#!/bin/bash
# round-2 GPU pass B: streaming attention A/B (bits), GPU suite, bench A/B
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_engine.py -q -s -x -k "streaming" -p no:cacheprovider > gpurun_out/r2b_stream_test.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_stream_test.log
timeout 900 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r2b_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_gputest.log
RLB_ATTN_STREAM=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2b_bench_k1.json 2> gpurun_out/r2b_bench_k1.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2b_bench_k1s.json 2> gpurun_out/r2b_bench_k1s.err
