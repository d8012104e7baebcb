#!/bin/bash
# final build: whole GPU suite, smoke, bench line
cd "$(dirname "$0")/.."
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2am_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/r2am_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2am_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r2am_smoke.log
timeout 900 python bench.py > gpurun_out/r2am_bench.json 2> gpurun_out/r2am_bench.err
