#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python scripts/ab_libs.py paper_2510_19225_b200/librlb.so paper_2510_19225_b200/librlb_p3b2.so paper_2510_19225_b200/librlb_n3b2.so > gpurun_out/r2k_ab.json 2>&1
for v in "" p3b2 n3b2; do
  lib=${v:+paper_2510_19225_b200/librlb_$v.so}
  RLB_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --steps 1 > gpurun_out/r2k_bench_${v:-base}.json 2>&1
  RLB_LIB=$lib timeout 900 python bench_migrate.py --instances 2 --kill 1 --prompts 256 > gpurun_out/r2k_migrate_${v:-base}.json 2>&1
done
