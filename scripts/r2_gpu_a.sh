#!/bin/bash
# round-2 GPU pass A: full GPU tests, bench, ncu of the profiled attention launch (mid + short context)
cd "$(dirname "$0")/.."
python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r2a_gputest.log 2>&1
echo "gputest rc=$?" >> gpurun_out/r2a_gputest.log
python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
for at in 0.5 0.1; do
  tag=$( [ "$at" = "0.5" ] && echo mid || echo short )
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:attn_mma -c 1 -f -o gpurun_out/r2_attn_$tag \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --profile-at $at \
    > gpurun_out/r2_attn_${tag}_bench.json 2> gpurun_out/r2_attn_${tag}.err
  python scripts/ncu_attn_json.py gpurun_out/r2_attn_$tag.ncu-rep gpurun_out/r2_attn_${tag}_bench.json \
    gpurun_out/r2_attn_${tag}_ncu.json > /dev/null 2>> gpurun_out/r2_attn_${tag}.err
done
