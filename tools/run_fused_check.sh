#!/bin/bash
# One-launch (fused) small-message path: emulated parity on GPU 0, real 2-GPU parity and timeout
# tests, then the message-size sweep with and without it.  Output under gpurun_out/fused/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/fused
export SDP4_WAIT_TIMEOUT_S=${SDP4_WAIT_TIMEOUT_S:-20}
timeout 900 python -m pytest tests/test_gpu_fused.py -x -q > gpurun_out/fused/emu.log 2>&1
echo "emu rc=$?" | tee -a gpurun_out/fused/summary.txt
tail -3 gpurun_out/fused/emu.log >> gpurun_out/fused/summary.txt
timeout 1200 python -m pytest tests/test_gpu_dist.py -x -q -k "not fullsize" > gpurun_out/fused/dist.log 2>&1
echo "dist rc=$?" | tee -a gpurun_out/fused/summary.txt
tail -3 gpurun_out/fused/dist.log >> gpurun_out/fused/summary.txt
n=$(python -c "import torch;print(torch.cuda.device_count())")
for lim in default 0; do
  extra=""; [ "$lim" = "0" ] && extra="--fused-limit 0"
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29650 + RANDOM % 200)) tools/size_sweep.py --graphs --sizes-mb ${SIZES:-1,4,16,64,256} $extra \
    --out gpurun_out/fused/sweep_n${n}_fused_${lim}.json > gpurun_out/fused/sweep_${lim}.log 2>&1
  echo "sweep $lim rc=$?" | tee -a gpurun_out/fused/summary.txt
done
cat gpurun_out/fused/summary.txt
