#!/bin/bash
# ncu --set full of the first prefill chunk's QKV (pairp<6>), O and down (pairp<7>) launches
cd "$(dirname "$0")/.."
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_pairp_tc<.int.[67]>" -c 3 \
  -o gpurun_out/r2ak_pairp python bench.py --steps 1 --warmup 0 --no-cpu-baseline --new-tokens 2 > gpurun_out/r2ak_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r2ak_ncu.log
