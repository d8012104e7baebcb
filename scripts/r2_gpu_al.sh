#!/bin/bash
# split-sum: h rows prefetched into L2 one unit before the last split
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_engine.py -m gpu -q -x -p no:cacheprovider -k "split_sum" > gpurun_out/r2al_test.log 2>&1
echo "rc=$?" >> gpurun_out/r2al_test.log
cp paper_2510_19225_b200/librlb.so /tmp/librlb_new.so
for r in 1 2; do
  RLB_LIB=paper_2510_19225_b200/librlb_base.so timeout 600 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/r2al_bench_base_$r.json 2>&1
  timeout 600 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/r2al_bench_new_$r.json 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|resid" \
  -c 400 --csv --log-file gpurun_out/r2al_launches_prefill.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --new-tokens 2 > /dev/null 2>&1
