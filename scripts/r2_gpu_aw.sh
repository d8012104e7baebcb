#!/bin/bash
# PDL mask around the new default 11: 3 (GEMM + attention), 9 (GEMM + small kernels)
cd "$(dirname "$0")/.."
b() { timeout 600 python bench.py --no-cpu-baseline --steps 2 "$@"; }
for r in 1 2; do
  b > gpurun_out/r2aw_m11_$r.json 2>&1
  RLB_PDL_MASK=3 b > gpurun_out/r2aw_m3_$r.json 2>&1
  RLB_PDL_MASK=9 b > gpurun_out/r2aw_m9_$r.json 2>&1
done
