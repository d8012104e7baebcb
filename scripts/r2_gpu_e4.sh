#!/bin/bash
# round-2 4-GPU pass: config 4 pulls (+ NVLink counters), config 5 with a late joiner,
# config 3 (8 instances, kill 2), bench at N=4
cd "$(dirname "$0")/.."
ncu --query-metrics 2>/dev/null | grep -i -E "nvl|ctc" > gpurun_out/r2e_ncu_nvl_metrics.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29511 bench_pull.py > gpurun_out/r2e_pull_1to3.json 2> gpurun_out/r2e_pull_1to3.err
timeout 1500 python bench_longtail.py --prompts 288 --max-inflight 384 --theta 32 --max-len 4096 \
  --late-join 256 --kv-gb 70 > gpurun_out/r2e_longtail.json 2> gpurun_out/r2e_longtail.err
timeout 900 python bench_migrate.py --instances 8 --kill 2 --check > gpurun_out/r2e_migrate8.json 2> gpurun_out/r2e_migrate8.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29512 bench.py --gpus 4 > gpurun_out/r2e_bench4.json 2> gpurun_out/r2e_bench4.err
# NVLink counters of the fused re-layout pull reading the 7B set over NVLink (single process, 2 GPUs)
for MET in "nvlrx__bytes.sum,nvltx__bytes.sum" "nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum" ""; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum${MET:+,$MET} \
    --clock-control none -k regex:chunk_copy -c 4 python scripts/peer_pull_probe.py --7b \
    > gpurun_out/r2e_ncu_k7.txt 2>&1 && grep -q "chunk_copy" gpurun_out/r2e_ncu_k7.txt && break
done
