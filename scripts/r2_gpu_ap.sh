#!/bin/bash
# decode attention ring depth (timing only): 3 stages (default) vs 2 at short and mid context
cd "$(dirname "$0")/.."
for at in 0.1 0.5; do
  for v in base s2 s2b6; do
    lib=paper_2510_19225_b200/librlb.so; [ $v != base ] && lib=paper_2510_19225_b200/librlb_$v.so
    RLB_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --steps 2 --profile-at $at > gpurun_out/r2ap_${v}_$at.json 2>&1
  done
done
