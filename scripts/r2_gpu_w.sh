#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn|gemm|resid|argmax|embed|seed|ring" \
  -c 1800 --csv --log-file gpurun_out/r2w_launches_prefill.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --new-tokens 2 > /dev/null 2>&1
