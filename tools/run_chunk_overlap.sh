#!/bin/bash
# P2P TLq-HS in chunks with K3 chained across chunks and capped to fewer SMs, so that K4/K5 of
# chunk k run beside the NVLink-bound K3 of chunk k+1 (4 GPUs, 2x2 and 4x1).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/chov
R() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) "$@"; }
B="bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --no-comparators --no-cpu-baseline --no-variants"
for g in 2 4; do
  R $B --groups $g > gpurun_out/chov/g${g}_c1.json 2>/dev/null; echo "g$g c1 rc=$?"
  for c in 2 3 4; do
    R $B --groups $g --chunks $c > gpurun_out/chov/g${g}_c${c}.json 2>/dev/null; echo "g$g c$c rc=$?"
    for k in 148 112 96; do
      SDP4_P2P_K3_CHAIN=1 SDP4_P2P_K3_SMS=$k R $B --groups $g --chunks $c > gpurun_out/chov/g${g}_c${c}_chain_k$k.json 2>/dev/null
      echo "g$g c$c chain k$k rc=$?"
    done
  done
done
