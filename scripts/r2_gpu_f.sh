#!/bin/bash
cd "$(dirname "$0")/.."
for v in "" s4b1 s5b1 s6b1; do
  lib=${v:+paper_2510_19225_b200/librlb_$v.so}
  RLB_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --steps 1 > gpurun_out/r2f_bench_${v:-base}.json 2>&1
  RLB_LIB=$lib RLB_ATTN_TMA=0 timeout 600 python bench.py --no-cpu-baseline --steps 1 > gpurun_out/r2f_bench_${v:-base}_cp.json 2>&1
done
