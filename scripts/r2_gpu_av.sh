#!/bin/bash
# confirm: RMSNorm kernels without PDL (RLB_PDL_MASK=11) vs all PDL
cd "$(dirname "$0")/.."
b() { timeout 600 python bench.py --no-cpu-baseline --steps 2 "$@"; }
for r in 1 2 3; do
  b > gpurun_out/r2av_base_$r.json 2>&1
  RLB_PDL_MASK=11 b > gpurun_out/r2av_m11_$r.json 2>&1
done
