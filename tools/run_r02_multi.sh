# Round-2 multi-GPU evidence on a 4-GPU box: distributed parity (real GPUs, both transports,
# graph replays, memop waits, bounded-wait timeout, bench-size windows), then the bench at
# 2 GPUs (2x1, 1x2) and 4 GPUs (2x2, 1x4, 4x1), then the message-size sweep at 2x2 and 1x4.
mkdir -p gpurun_out/multi
python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/multi/pytest_dist.log 2>&1; tail -2 gpurun_out/multi/pytest_dist.log
R() { n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) "$@"; }
summ() { python -c "
import json,sys
d=json.loads(open('$1').read().strip().splitlines()[-1]); c=d.get('comparators') or {}
print(d['config']['workload'], 'ms', d['ms_per_step'], 'GB/s', d['value'], 'e2e', (d.get('e2e') or {}).get('value'), 'lfl', c.get('like_for_like'), {n:(v['avg_ms'], v.get('nvlink_gbs')) for n,v in d['kernels'].items()})" 2>/dev/null || tail -3 ${1%.json}.err; }
CUDA_VISIBLE_DEVICES=0,1 R 2 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/multi/bench_n2_2x1.json 2> gpurun_out/multi/bench_n2_2x1.err; summ gpurun_out/multi/bench_n2_2x1.json
CUDA_VISIBLE_DEVICES=0,1 R 2 bench.py --gpus 2 --steps 20 --warmup 5 --groups 1 --no-e2e > gpurun_out/multi/bench_n2_1x2.json 2> gpurun_out/multi/bench_n2_1x2.err; summ gpurun_out/multi/bench_n2_1x2.json
R 4 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/multi/bench_n4_2x2.json 2> gpurun_out/multi/bench_n4_2x2.err; summ gpurun_out/multi/bench_n4_2x2.json
R 4 bench.py --gpus 4 --steps 20 --warmup 5 --groups 1 --no-e2e > gpurun_out/multi/bench_n4_1x4.json 2> gpurun_out/multi/bench_n4_1x4.err; summ gpurun_out/multi/bench_n4_1x4.json
R 4 bench.py --gpus 4 --steps 20 --warmup 5 --groups 4 --no-e2e > gpurun_out/multi/bench_n4_4x1.json 2> gpurun_out/multi/bench_n4_4x1.err; summ gpurun_out/multi/bench_n4_4x1.json
R 4 tools/size_sweep.py --graphs --out gpurun_out/multi/size_sweep_n4_2x2.json > gpurun_out/multi/size_2x2.log 2>&1; tail -2 gpurun_out/multi/size_2x2.log
R 4 tools/size_sweep.py --graphs --groups 1 --out gpurun_out/multi/size_sweep_n4_1x4.json > gpurun_out/multi/size_1x4.log 2>&1; tail -2 gpurun_out/multi/size_1x4.log
