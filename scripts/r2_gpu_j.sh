#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1800 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r2j_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/r2j_gputest.log
timeout 600 python bench.py > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn|gemm|resid|argmax|embed|decode_prepare" \
  --launch-skip 6000 -c 600 --csv --log-file gpurun_out/r2j_launches_decode.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
