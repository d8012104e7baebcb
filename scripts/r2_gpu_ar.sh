#!/bin/bash
# ncu --set full of one decode layer's GEMMs and RMSNorms (final build)
cd "$(dirname "$0")/.."
timeout 1500 ncu --set full --clock-control none -k regex:"gemm|resid" --launch-skip 3000 -c 8 \
  -o gpurun_out/r2ar_decode python bench.py --steps 1 --warmup 0 --no-cpu-baseline --new-tokens 64 > gpurun_out/r2ar_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r2ar_ncu.log
