#!/bin/bash
# decode down projection plans (numerics plan: split factor; tile/reduction modes keep bits)
cd "$(dirname "$0")/.."
b() { timeout 600 python bench.py --no-cpu-baseline --steps 2 "$@"; }
b > gpurun_out/r2ah_base.json 2>&1
b --split-down 6 > gpurun_out/r2ah_sd6.json 2>&1
RLB_PAIRP=26 b --split-down 3 > gpurun_out/r2ah_cl_sd3.json 2>&1
RLB_PAIRP=26 RLB_CLUSTER=0,0 b --split-down 3 > gpurun_out/r2ah_part_sd3.json 2>&1
RLB_PAIRP=26 b --split-down 5 > gpurun_out/r2ah_cl_sd5.json 2>&1
RLB_PAIRP=26 b --split-down 4 > gpurun_out/r2ah_cl_sd4.json 2>&1
b --split-down 7 > gpurun_out/r2ah_sd7.json 2>&1
