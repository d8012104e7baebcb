#!/bin/bash
# prefill groups (K1g): bits A/B, suite, bench A/B, 1-GPU resume A/B, prefill launch list
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_engine.py -q -s -x -k "groups_same_bits" -p no:cacheprovider > gpurun_out/r2g_groups_test.log 2>&1
echo "rc=$?" >> gpurun_out/r2g_groups_test.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2g_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/r2g_gputest.log
RLB_ATTN_GROUPS=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2g_bench_pairs.json 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2g_bench_groups.json 2>&1
RLB_ATTN_GROUPS=0 timeout 900 python bench_migrate.py --instances 2 --kill 1 --prompts 256 > gpurun_out/r2g_migrate_pairs.json 2>&1
timeout 900 python bench_migrate.py --instances 2 --kill 1 --prompts 256 --check > gpurun_out/r2g_migrate_groups.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file gpurun_out/r2g_launches_prefill.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --new-tokens 2 > /dev/null 2>&1
