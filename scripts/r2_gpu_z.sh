#!/bin/bash
# A/B: epilogue of the fp32 partial tiles on 8 warps (librlb.so) vs 4 (librlb_base.so)
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2z_test.log 2>&1
echo "rc=$?" >> gpurun_out/r2z_test.log
timeout 600 python scripts/ab_libs.py paper_2510_19225_b200/librlb_base.so paper_2510_19225_b200/librlb.so > gpurun_out/r2z_ab.log 2>&1
for r in 1 2; do
  for v in base new; do
    lib=paper_2510_19225_b200/librlb.so; [ $v = base ] && lib=paper_2510_19225_b200/librlb_base.so
    RLB_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/r2z_bench_${v}_$r.json 2>&1
  done
done
for v in base new; do
  lib=paper_2510_19225_b200/librlb.so; [ $v = base ] && lib=paper_2510_19225_b200/librlb_base.so
  RLB_LIB=$lib timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm" \
    --launch-skip 3000 -c 400 --csv --log-file gpurun_out/r2z_launches_$v.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
done
