#!/bin/bash
# final-default pass: GPU suite, smoke, bench, ncu of the profiled attention launch (mid + short)
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r2r_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/r2r_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2r_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_smoke.log
timeout 600 python bench.py > gpurun_out/r2r_bench.json 2> gpurun_out/r2r_bench.err
for at in 0.5 0.1; do
  tag=$( [ "$at" = "0.5" ] && echo mid || echo short )
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:attn_mma -c 1 -f -o gpurun_out/r2r_attn_$tag \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --profile-at $at \
    > gpurun_out/r2r_attn_${tag}_bench.json 2> gpurun_out/r2r_attn_${tag}.err
done
