#!/bin/bash
# decode attention window length (numerics plan 'w'): 2048 (default) vs 1024 / 512 positions per CTA
cd "$(dirname "$0")/.."
for r in 1 2; do
  for v in base w1024 w512; do
    lib=paper_2510_19225_b200/librlb.so; [ $v != base ] && lib=paper_2510_19225_b200/librlb_$v.so
    RLB_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/r2ai_${v}_$r.json 2>&1
  done
done
