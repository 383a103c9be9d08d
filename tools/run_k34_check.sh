#!/bin/bash
# K34 (N = 1 fused K3 + K4): shared-GPU parity (all splits), real 2-GPU parity, 2-GPU bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/k34
export SDP4_WAIT_TIMEOUT_S=20
timeout 1200 python -m pytest tests/test_gpu_virtual.py -x -q -k "all_splits" > gpurun_out/k34/virtual.log 2>&1
echo "virtual rc=$?"; tail -1 gpurun_out/k34/virtual.log
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q -k "not fullsize" > gpurun_out/k34/dist.log 2>&1
echo "dist rc=$?"; tail -1 gpurun_out/k34/dist.log
for g in 2 1; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700 + g)) bench.py --gpus 2 --groups $g > gpurun_out/k34/bench_n2_g$g.json 2> gpurun_out/k34/bench_n2_g$g.err
  echo "bench g=$g rc=$?"
done
