#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2l_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_smoke.log
timeout 900 python bench_migrate.py --check > gpurun_out/r2l_migrate4.json 2> gpurun_out/r2l_migrate4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29513 bench.py --gpus 2 > gpurun_out/r2l_bench2.json 2> gpurun_out/r2l_bench2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29514 bench.py --gpus 4 --strong > gpurun_out/r2l_bench4_strong.json 2> gpurun_out/r2l_bench4_strong.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29515 bench_pull.py > gpurun_out/r2l_pull_1to1.json 2> gpurun_out/r2l_pull_1to1.err
