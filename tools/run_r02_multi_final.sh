#!/bin/bash
# Round-2 multi-GPU evidence on a 4-GPU box (final kernels): distributed parity on real GPUs,
# the bench at 2 GPUs (2x1, 1x2) and 4 GPUs (2x2, 1x4, 4x1), the message-size sweeps.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/multi
timeout 1500 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/multi/pytest_dist.log 2>&1; echo "dist rc=$?"; tail -1 gpurun_out/multi/pytest_dist.log
R() { n=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) "$@"; }
CUDA_VISIBLE_DEVICES=0,1 R 2 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/multi/bench_n2_2x1.json 2> gpurun_out/multi/bench_n2_2x1.err; echo "n2 2x1 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 R 2 bench.py --gpus 2 --steps 20 --warmup 5 --groups 1 --no-e2e > gpurun_out/multi/bench_n2_1x2.json 2> gpurun_out/multi/bench_n2_1x2.err; echo "n2 1x2 rc=$?"
R 4 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/multi/bench_n4_2x2.json 2> gpurun_out/multi/bench_n4_2x2.err; echo "n4 2x2 rc=$?"
R 4 bench.py --gpus 4 --steps 20 --warmup 5 --groups 1 --no-e2e > gpurun_out/multi/bench_n4_1x4.json 2> gpurun_out/multi/bench_n4_1x4.err; echo "n4 1x4 rc=$?"
R 4 bench.py --gpus 4 --steps 20 --warmup 5 --groups 4 --no-e2e > gpurun_out/multi/bench_n4_4x1.json 2> gpurun_out/multi/bench_n4_4x1.err; echo "n4 4x1 rc=$?"
bash tools/run_r02_sizes_fused.sh
