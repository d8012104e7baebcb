#!/bin/bash
# final-build 1-GPU evidence: smoke, bench line (with CPU baseline), reference arm,
# decode + prefill launch lists
cd "$(dirname "$0")/.."
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ae_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r2ae_smoke.log
timeout 900 python bench.py > gpurun_out/r2ae_bench.json 2> gpurun_out/r2ae_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2ae_ref.json 2> gpurun_out/r2ae_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn|gemm|resid|argmax|embed|decode_prepare" \
  --launch-skip 6000 -c 600 --csv --log-file gpurun_out/r2ae_launches_decode.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn|gemm|resid|argmax|embed|seed|ring" \
  -c 1800 --csv --log-file gpurun_out/r2ae_launches_prefill.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --new-tokens 2 > /dev/null 2>&1
