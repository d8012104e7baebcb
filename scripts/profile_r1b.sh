#!/bin/bash
# Round-1 refresh after the 2-SM split-K down projection (run via gpurun, 1 GPU).
set -e
OUT=${OUT:-gpurun_out}
# the committed bench line: default arguments (N=1, CPU baseline included)
python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > $OUT/plain.json 2> $OUT/plain.err
ncu --metrics gpu__time_duration.sum --clock-control none -s 150000 -c 600 --csv \
    --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2400 --csv \
    --log-file $OUT/launches_prefill.csv $CMD > $OUT/ncu_launch_prefill.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_pairp -s 3000 -c 2 \
    -o $OUT/prof_pairp $CMD > $OUT/ncu_pairp.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_pair -s 20 -c 1 \
    -o $OUT/prof_attn_pair $CMD > $OUT/ncu_attn_pair.log 2>&1
for r in prof_pairp prof_attn_pair; do
  python scripts/ncu_summary.py $OUT/$r.ncu-rep > $OUT/$r.summary.txt
  ncu -i $OUT/$r.ncu-rep --page details --csv > $OUT/$r.details.csv
  rm -f $OUT/$r.ncu-rep || true
done
echo profile-done
