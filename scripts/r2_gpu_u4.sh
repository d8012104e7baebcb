#!/bin/bash
# final-build multi-GPU pass
cd "$(dirname "$0")/.."
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29521 bench.py --gpus 4 > gpurun_out/r2u_bench4.json 2> gpurun_out/r2u_bench4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29522 bench.py --gpus 2 > gpurun_out/r2u_bench2.json 2> gpurun_out/r2u_bench2.err
timeout 900 python bench_migrate.py --instances 8 --kill 2 --check > gpurun_out/r2u_migrate8.json 2> gpurun_out/r2u_migrate8.err
CUDA_VISIBLE_DEVICES=0,1 timeout 1500 python bench_longtail.py --instances 2 --prompts 192 --max-inflight 384 --theta 32 \
  --max-len 4096 --late-join 256 --kv-gb 70 > gpurun_out/r2u_longtail2.json 2> gpurun_out/r2u_longtail2.err
