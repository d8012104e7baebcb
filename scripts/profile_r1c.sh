#!/bin/bash
# Round-1 final refresh (run via gpurun, 1 GPU): bench line, decode launch
# list, ncu --set full of the QKV (3D-box stages) and down (2-SM pair) GEMMs.
set -e
OUT=${OUT:-gpurun_out}
python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -s 150000 -c 600 --csv \
    --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_tc -s 4000 -c 5 \
    -o $OUT/prof_gemm $CMD > $OUT/ncu_gemm.log 2>&1
python scripts/ncu_summary.py $OUT/prof_gemm.ncu-rep > $OUT/prof_gemm.summary.txt
rm -f $OUT/prof_gemm.ncu-rep || true
echo profile-done
