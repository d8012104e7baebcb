#!/bin/bash
# compute-sanitizer over the tiny-shape GPU tests (memcheck, racecheck, synccheck, initcheck)
cd "$(dirname "$0")/.."
SEL='tests/test_gpu_engine.py::test_tiny_rollout_teacher_forced tests/test_gpu_engine.py::test_tiny_score_logits tests/test_gpu_engine.py::test_tiny_migration_bit_exact tests/test_gpu_kernels.py'
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 \
    --log-file gpurun_out/r2_san_$tool.txt \
    python -m pytest $SEL -q -p no:cacheprovider > gpurun_out/r2_san_${tool}_pytest.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r2_san_summary.txt
  tail -3 gpurun_out/r2_san_$tool.txt >> gpurun_out/r2_san_summary.txt
done
