#!/bin/bash
cd "$(dirname "$0")/.."
for v in "" w2 w2s4 w1 w1s4 w2p3; do
  lib=${v:+paper_2510_19225_b200/librlb_$v.so}
  RLB_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/r2q_bench_${v:-base}.json 2>&1
done
for v in w2 w1 w2p3; do
  RLB_LIB=paper_2510_19225_b200/librlb_$v.so timeout 900 python bench_migrate.py --instances 2 --kill 1 --prompts 256 > gpurun_out/r2q_migrate_$v.json 2>&1
done
