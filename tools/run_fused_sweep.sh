#!/bin/bash
# Message-size sweep with the one-launch path forced on and off.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/fused
n=$(python -c "import torch;print(torch.cuda.device_count())")
G=${GROUPS_ARG:-}
for lim in 1000000000 0; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29650 + RANDOM % 200)) tools/size_sweep.py --graphs --sizes-mb ${SIZES:-1,2,4,8,16,32,64,128,256} \
    --fused-limit $lim $G --out gpurun_out/fused/sweep_n${n}${TAG}_lim${lim}.json > gpurun_out/fused/sweep_n${n}${TAG}_lim${lim}.log 2>&1
  echo "sweep n=$n lim=$lim rc=$?"
done
