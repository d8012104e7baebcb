#!/bin/bash
# round-2 GPU pass D: TMA decode attention A/B (bits), GPU suite, bench A/B
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_engine.py -q -s -x -k "tma_same_bits" -p no:cacheprovider > gpurun_out/r2d_tma_test.log 2>&1
echo "rc=$?" >> gpurun_out/r2d_tma_test.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2d_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/r2d_gputest.log
RLB_ATTN_TMA=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2d_bench_cpasync.json 2> gpurun_out/r2d_bench_cpasync.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2d_bench_tma.json 2> gpurun_out/r2d_bench_tma.err
