#!/bin/bash
# K34 with the 4-bit group max taken from the 8-bit step: parity (emulated M x 1 nodes, shared-GPU
# 2-rank splits incl. 2x1) and timing (tools/k34_probe.py, before/after in the log).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/k34f
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py -q -x > gpurun_out/k34f/parity.log 2>&1
echo "parity rc=$?"; tail -1 gpurun_out/k34f/parity.log
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x -k "all_splits and 2" > gpurun_out/k34f/virtual.log 2>&1
echo "virtual rc=$?"; tail -1 gpurun_out/k34f/virtual.log
for i in 1 2 3; do python tools/k34_probe.py; done > gpurun_out/k34f/probe.log 2>&1
cat gpurun_out/k34f/probe.log
