#!/bin/bash
cd "$(dirname "$0")/.."
for v in "" w2; do
  lib=${v:+paper_2510_19225_b200/librlb_$v.so}
  RLB_LIB=$lib timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2p_bench_${v:-base}.json 2>&1
  RLB_LIB=$lib timeout 900 python bench_migrate.py --instances 2 --kill 1 --prompts 256 > gpurun_out/r2p_migrate_${v:-base}.json 2>&1
done
RLB_LIB=paper_2510_19225_b200/librlb_w2.so timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider \
  --deselect tests/test_gpu_checked.py::test_engine_suite_on_checked_build > gpurun_out/r2p_gputest_w2.log 2>&1
echo "rc=$?" >> gpurun_out/r2p_gputest_w2.log
