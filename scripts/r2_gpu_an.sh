#!/bin/bash
# decode QKV (64-column RoPE tiles): epilogue on 8 warps (16-column halves) vs 4
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2an_test.log 2>&1
echo "rc=$?" >> gpurun_out/r2an_test.log
timeout 600 python scripts/ab_libs.py paper_2510_19225_b200/librlb_base.so paper_2510_19225_b200/librlb.so > gpurun_out/r2an_ab.log 2>&1
for r in 1 2; do
  RLB_LIB=paper_2510_19225_b200/librlb_base.so timeout 600 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/r2an_bench_base_$r.json 2>&1
  timeout 600 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/r2an_bench_new_$r.json 2>&1
done
