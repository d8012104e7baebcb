#!/bin/bash
# split-sum epilogue (EPI_SUMRES) for prefill O / down: bits, A/B, launch list
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_kernels.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2aa_test.log 2>&1
echo "rc=$?" >> gpurun_out/r2aa_test.log
timeout 600 python scripts/ab_libs.py paper_2510_19225_b200/librlb_base.so paper_2510_19225_b200/librlb.so > gpurun_out/r2aa_ab.log 2>&1
for r in 1 2; do
  RLB_SUMRES=0 timeout 600 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/r2aa_bench_off_$r.json 2>&1
  timeout 600 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/r2aa_bench_on_$r.json 2>&1
done
timeout 600 python bench.py --no-cpu-baseline --steps 2 --prefill-rows 18944 > gpurun_out/r2aa_bench_on_18944.json 2>&1
RLB_SUMRES=0 timeout 600 python bench.py --no-cpu-baseline --steps 2 --prefill-rows 18944 > gpurun_out/r2aa_bench_off_18944.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn|gemm|resid|argmax|embed|seed|ring" \
  -c 1800 --csv --log-file gpurun_out/r2aa_launches_prefill.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --new-tokens 2 > /dev/null 2>&1
