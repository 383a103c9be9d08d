#!/bin/bash
# K345 (world 1) with the known 4-bit max: parity and the one-GPU bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/k345
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_determinism.py -q -x > gpurun_out/k345/parity.log 2>&1
echo "parity rc=$?"; tail -1 gpurun_out/k345/parity.log
for i in 1 2; do python bench.py --no-e2e --no-cpu-baseline > gpurun_out/k345/bench_$i.json 2>/dev/null; echo "bench rc=$?"; done
