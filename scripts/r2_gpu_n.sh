#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_engine.py -q -s -x -k "head16_same_bits" -p no:cacheprovider > gpurun_out/r2n_head16_test.log 2>&1
echo "rc=$?" >> gpurun_out/r2n_head16_test.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2n_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/r2n_gputest.log
for f in 0 1; do
  RLB_ATTN_HEAD16=$f timeout 600 python bench.py --no-cpu-baseline --steps 1 > gpurun_out/r2n_bench_h$f.json 2>&1
  RLB_ATTN_HEAD16=$f timeout 900 python bench_migrate.py --instances 2 --kill 1 --prompts 256 > gpurun_out/r2n_migrate_h$f.json 2>&1
done
