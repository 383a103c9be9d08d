#!/bin/bash
# Message-size sweeps (BASELINE config 5) with the library defaults (one-launch path below
# its limits): 4 GPUs 2x2 / 1x4 / 4x1 -> gpurun_out/multi/size_sweep_n4_*.json.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/multi
n=$(python -c "import torch;print(torch.cuda.device_count())")
for g in ${SPLITS:-2 1 4}; do
  M=$g; N=$((n / g))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 300)) tools/size_sweep.py --graphs --groups $g \
    --out gpurun_out/multi/size_sweep_n${n}_${M}x${N}.json > gpurun_out/multi/size_${M}x${N}.log 2>&1
  echo "split ${M}x${N} rc=$?"
done
