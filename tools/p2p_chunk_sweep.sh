mkdir -p gpurun_out/p2pc
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for g in 2 1; do for c in 1 2 3 4; do tag=g${g}_c$c
$R --master-port 29$((RANDOM%800+100)) bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-comparators --groups $g --chunks $c > gpurun_out/p2pc/$tag.json 2> gpurun_out/p2pc/$tag.err
python -c "
import json; d=json.loads(open('gpurun_out/p2pc/$tag.json').read().splitlines()[-1]); print('$tag', d['ms_per_step'], 'tlq', d['collectives']['tlq_hs_reduce_scatter']['ms'], {n[:2]: v['avg_ms'] for n,v in d['kernels'].items()})" || tail -3 gpurun_out/p2pc/$tag.err
done; done
