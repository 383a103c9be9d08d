#!/bin/bash
# Bench lines of the splits that run K34 (2x1 on 2 GPUs, 4x1 on 4 GPUs) after the known-max change.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/multi
R() { n=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) "$@"; }
CUDA_VISIBLE_DEVICES=0,1 R 2 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/multi/bench_n2_2x1.json 2> gpurun_out/multi/bench_n2_2x1.err; echo "n2 2x1 rc=$?"
R 4 bench.py --gpus 4 --steps 20 --warmup 5 --groups 4 --no-e2e > gpurun_out/multi/bench_n4_4x1.json 2> gpurun_out/multi/bench_n4_4x1.err; echo "n4 4x1 rc=$?"
