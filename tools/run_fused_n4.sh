#!/bin/bash
# 4 GPUs: multi-GPU parity (incl. the one-launch path) + fused on/off sweeps for 2x2, 1x4, 4x1.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/fused
export SDP4_WAIT_TIMEOUT_S=20
timeout 1500 python -m pytest tests/test_gpu_dist.py -x -q -k "not fullsize" > gpurun_out/fused/dist_n4.log 2>&1
echo "dist rc=$?"; tail -2 gpurun_out/fused/dist_n4.log
for g in 2 1 4; do
  GROUPS_ARG="--groups $g" TAG="_g$g" SIZES=${SIZES:-1,4,16,32,64} bash tools/run_fused_sweep.sh
done
