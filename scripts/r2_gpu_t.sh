#!/bin/bash
cd "$(dirname "$0")/.."
for v in "" w2s2 w2s2b5; do
  lib=${v:+paper_2510_19225_b200/librlb_$v.so}
  RLB_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/r2t_bench_${v:-base}.json 2>&1
  RLB_LIB=$lib RLB_ATTN_TMA=0 timeout 600 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/r2t_bench_${v:-base}_cp.json 2>&1
done
