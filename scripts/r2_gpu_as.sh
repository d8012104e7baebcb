#!/bin/bash
# decode gate_up as two 256 x 128 SwiGLU CTAs per SM (RLB_GU2=1) vs one 256 x 256 CTA
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_engine.py -m gpu -q -x -p no:cacheprovider -k "parity or migration" > gpurun_out/r2as_test.log 2>&1
echo "rc=$?" >> gpurun_out/r2as_test.log
RLB_GU2=1 timeout 900 python -m pytest tests/test_gpu_engine.py -m gpu -q -x -p no:cacheprovider -k "parity or migration" > gpurun_out/r2as_test_gu2.log 2>&1
echo "rc=$?" >> gpurun_out/r2as_test_gu2.log
for r in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/r2as_bench_base_$r.json 2>&1
  RLB_GU2=1 timeout 600 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/r2as_bench_gu2_$r.json 2>&1
done
