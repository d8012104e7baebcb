#!/bin/bash
# split-sum with the running sum in TMEM for O: bits, A/B, prefill launch list
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_engine.py -m gpu -q -x -p no:cacheprovider -k "split_sum" > gpurun_out/r2af_test.log 2>&1
echo "rc=$?" >> gpurun_out/r2af_test.log
timeout 600 python scripts/ab_libs.py paper_2510_19225_b200/librlb_base.so paper_2510_19225_b200/librlb.so > gpurun_out/r2af_ab.log 2>&1
for r in 1 2; do
  RLB_SUMRES_TMEM=0 timeout 600 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/r2af_bench_l2_$r.json 2>&1
  timeout 600 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/r2af_bench_tmem_$r.json 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|resid" \
  -c 400 --csv --log-file gpurun_out/r2af_launches_prefill.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --new-tokens 2 > /dev/null 2>&1
