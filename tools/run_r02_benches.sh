#!/bin/bash
# Final multi-GPU bench lines (4-GPU box): 2 GPUs (2x1, 1x2), 4 GPUs (2x2, 1x4, 4x1).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/multi
R() { n=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) "$@"; }
CUDA_VISIBLE_DEVICES=0,1 R 2 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/multi/bench_n2_2x1.json 2> gpurun_out/multi/bench_n2_2x1.err; echo "n2 2x1 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 R 2 bench.py --gpus 2 --steps 20 --warmup 5 --groups 1 --no-e2e > gpurun_out/multi/bench_n2_1x2.json 2> gpurun_out/multi/bench_n2_1x2.err; echo "n2 1x2 rc=$?"
R 4 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/multi/bench_n4_2x2.json 2> gpurun_out/multi/bench_n4_2x2.err; echo "n4 2x2 rc=$?"
R 4 bench.py --gpus 4 --steps 20 --warmup 5 --groups 1 --no-e2e > gpurun_out/multi/bench_n4_1x4.json 2> gpurun_out/multi/bench_n4_1x4.err; echo "n4 1x4 rc=$?"
R 4 bench.py --gpus 4 --steps 20 --warmup 5 --groups 4 --no-e2e > gpurun_out/multi/bench_n4_4x1.json 2> gpurun_out/multi/bench_n4_4x1.err; echo "n4 4x1 rc=$?"
