#!/bin/bash
# prefill/decode projection mode sweep (tile / reduction modes: same bits)
cd "$(dirname "$0")/.."
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --steps 1 > gpurun_out/r2s_$tag.json 2>&1; }
run base X=1
run o_cluster RLB_PAIRP=22 RLB_CLUSTER=1,1
run o_single RLB_PAIRP=22
run down_cluster_large RLB_PAIRP=26 RLB_CLUSTER=0,1,1
run down_single RLB_PAIRP=26
run qkv_single RLB_PAIRP=14
