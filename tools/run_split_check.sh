#!/bin/bash
# One-launch TLq-HS phase C with split rows: 1-GPU emulated parity, real 4-GPU parity of the
# one-launch path, the 2x2 phase trace and the small-size sweep (gpurun --gpus 4).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/split
export SDP4_WAIT_TIMEOUT_S=20
timeout 900 python -m pytest tests/test_gpu_fused.py -x -q > gpurun_out/split/fused_1gpu.log 2>&1
echo "fused rc=$?"; tail -1 gpurun_out/split/fused_1gpu.log
n=$(python -c "import torch;print(torch.cuda.device_count())")
if [ "$n" -ge 2 ]; then
  timeout 1200 python -m pytest tests/test_gpu_dist.py -x -q -k "not fullsize" > gpurun_out/split/dist.log 2>&1
  echo "dist rc=$?"; tail -1 gpurun_out/split/dist.log
  SDP4_FUSED_TRACE=1 TRACE_MB=1,4,16 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port 29655 tools/fused_trace.py > gpurun_out/split/trace.log 2>&1
  echo "trace rc=$?"
  for g in ${SPLITS:-2}; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29600 + RANDOM % 300)) tools/size_sweep.py --groups $g --sizes-mb ${SIZES:-1,2,4,8,16,32,64} \
      --out gpurun_out/split/sweep_g$g.json > gpurun_out/split/sweep_g$g.log 2>&1
    echo "sweep g$g rc=$?"
  done
fi
