#!/bin/bash
# tile choice by work per SM (RLB_TILE_COST=1) vs fewest waves, decode profiles of both shapes
cd "$(dirname "$0")/.."
B=192,256,320,384,448,512
for r in 1 2; do
  timeout 600 python scripts/decode_profile.py gpurun_out/r2aj_7b_base_$r.json --shape qwen2.5-7b --batches $B > /dev/null 2>&1
  RLB_TILE_COST=1 timeout 600 python scripts/decode_profile.py gpurun_out/r2aj_7b_cost_$r.json --shape qwen2.5-7b --batches $B > /dev/null 2>&1
  timeout 600 python scripts/decode_profile.py gpurun_out/r2aj_15b_base_$r.json --batches $B > /dev/null 2>&1
  RLB_TILE_COST=1 timeout 600 python scripts/decode_profile.py gpurun_out/r2aj_15b_cost_$r.json --batches $B > /dev/null 2>&1
done
