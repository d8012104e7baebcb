#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_parity_full.py -q -s -p no:cacheprovider > gpurun_out/r2m_parity.log 2>&1
echo "rc=$?" >> gpurun_out/r2m_parity.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29516 bench_pull.py > gpurun_out/r2m_pull_1to1.json 2> gpurun_out/r2m_pull_1to1.err
