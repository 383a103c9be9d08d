# Round-2 BASELINE configs 3-4 and the qWD G=2048 row with the current
# kernels: GPT-6.7B at 1 GPU and 2x2 / 4x1 / 1x4; GPT-13B at 2 GPUs (2x1, 1x2) and 4 GPUs (2x2)
# with G in {64, 128, 256}; GPT-1.3B with G in {64, 256} and qWD at G_w = 2048 at 1 and 4 GPUs.
# GPT-13B at 1 GPU: with the world-1 fused TLq-HS kernel (no 20 GB of 8- / 4-bit workspace)
# the step needs ~161 GB of the 179 GB.
mkdir -p gpurun_out/cfg
R() { n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) "$@"; }
summ() { python -c "
import json,sys
d=json.loads(open('$1').read().strip().splitlines()[-1]); c=d.get('comparators') or {}
print(d['config']['workload'], 'ms', d['ms_per_step'], 'GB/s', d['value'], 'lfl', c.get('like_for_like'), {n:v['avg_ms'] for n,v in d['kernels'].items()})" 2>/dev/null || tail -3 ${1%.json}.err; }
export PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True
one() { name=$1; shift; CUDA_VISIBLE_DEVICES=0 python bench.py "$@" > gpurun_out/cfg/$name.json 2> gpurun_out/cfg/$name.err; summ gpurun_out/cfg/$name.json; }
many() { n=$1; name=$2; shift 2; R $n bench.py --gpus $n "$@" > gpurun_out/cfg/$name.json 2> gpurun_out/cfg/$name.err; summ gpurun_out/cfg/$name.json; }
one n1_1.3B_G64 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --group 64 --qwd-group 64
one n1_1.3B_G256 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --group 256 --qwd-group 256
one n1_1.3B_Gw2048 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --qwd-group 2048
one n1_6.7B --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --model 6.7B
one n1_13B --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-comparators --no-variants --model 13B
many 4 n4_1.3B_G64 --steps 10 --warmup 3 --no-e2e --group 64 --qwd-group 64
many 4 n4_1.3B_G256 --steps 10 --warmup 3 --no-e2e --group 256 --qwd-group 256
many 4 n4_1.3B_Gw2048 --steps 10 --warmup 3 --no-e2e --qwd-group 2048
many 4 n4_6.7B_2x2 --steps 10 --warmup 3 --no-e2e --model 6.7B
many 4 n4_6.7B_4x1 --steps 10 --warmup 3 --no-e2e --no-comparators --no-variants --model 6.7B --groups 4
many 4 n4_6.7B_1x4 --steps 10 --warmup 3 --no-e2e --no-comparators --no-variants --model 6.7B --groups 1
for G in 64 128 256; do many 4 n4_13B_2x2_G$G --steps 5 --warmup 3 --no-e2e --no-comparators --no-variants --model 13B --group $G --qwd-group $G; done
CUDA_VISIBLE_DEVICES=0,1 many 2 n2_13B_2x1 --steps 5 --warmup 3 --no-e2e --no-comparators --no-variants --model 13B
CUDA_VISIBLE_DEVICES=0,1 many 2 n2_13B_1x2 --steps 5 --warmup 3 --no-e2e --no-comparators --no-variants --model 13B --groups 1
