#!/bin/bash
# ncu evidence for the bench (run on the GPU box via gpurun, 1 GPU).
#   1. plain bench run (must exit 0 before any ncu run)
#   2. launch list mid-rollout: per-kernel device time (cold-cache, serialised)
#   3. --set full on the top kernels (attention, GEMMs)
set -e
OUT=${OUT:-gpurun_out}
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
# the same command as the bench line minus the CPU baseline (the launch list is a share check)
$CMD > $OUT/plain.json 2> $OUT/plain.err
ncu --metrics gpu__time_duration.sum --clock-control none -s 150000 -c 600 --csv \
    --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
# prefill: the first launches of the first rollout (weight load + varlen prefill chunks)
ncu --metrics gpu__time_duration.sum --clock-control none -c 2400 --csv \
    --log-file $OUT/launches_prefill.csv $CMD > $OUT/ncu_launch_prefill.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_mma -s 3000 -c 2 \
    -o $OUT/prof_attn $CMD > $OUT/ncu_attn.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 4000 -c 5 \
    -o $OUT/prof_gemm $CMD > $OUT/ncu_gemm.log 2>&1
echo profile-done
