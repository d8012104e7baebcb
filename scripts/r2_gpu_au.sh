#!/bin/bash
# launch-level knobs on the final build: PDL per kernel class, graph length
cd "$(dirname "$0")/.."
b() { timeout 600 python bench.py --no-cpu-baseline --steps 2 "$@"; }
for r in 1 2; do
  b > gpurun_out/r2au_base_$r.json 2>&1
  RLB_PDL_MASK=13 b > gpurun_out/r2au_nopdl_attn_$r.json 2>&1      # attention without PDL
  RLB_PDL_MASK=11 b > gpurun_out/r2au_nopdl_norm_$r.json 2>&1      # RMSNorm without PDL
  RLB_GRAPH_STEPS=32 b > gpurun_out/r2au_g32_$r.json 2>&1
done
RLB_NO_PDL=1 b > gpurun_out/r2au_nopdl_1.json 2>&1
