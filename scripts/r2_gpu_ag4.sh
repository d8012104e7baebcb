#!/bin/bash
# final-build multi-GPU pass (split-sum prefill): config-3 resume (4 and 8 instances), weak scaling 2 / 4
cd "$(dirname "$0")/.."
timeout 900 python bench_migrate.py --check > gpurun_out/r2ag_migrate4.json 2> gpurun_out/r2ag_migrate4.err
timeout 900 python bench_migrate.py --instances 8 --kill 2 --check > gpurun_out/r2ag_migrate8.json 2> gpurun_out/r2ag_migrate8.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29531 bench.py --gpus 4 > gpurun_out/r2ag_bench4.json 2> gpurun_out/r2ag_bench4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29532 bench.py --gpus 2 > gpurun_out/r2ag_bench2.json 2> gpurun_out/r2ag_bench2.err
