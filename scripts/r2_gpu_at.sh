#!/bin/bash
# decode O / QKV ring depth (timing only): 3 / 4 stages (default) vs 2 -- smaller smem lets the
# next GEMM's CTA start beside the draining attention / RMSNorm CTAs
cd "$(dirname "$0")/.."
for r in 1 2; do
  for v in base o2 q2 oq2; do
    lib=paper_2510_19225_b200/librlb.so; [ $v != base ] && lib=paper_2510_19225_b200/librlb_$v.so
    RLB_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/r2at_${v}_$r.json 2>&1
  done
done
