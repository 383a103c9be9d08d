# usage: bash tools/pull_sweep.sh NGPUS "groups ..." "splits ..."  -- push/pull split of the P2P intra all-to-all
N=${1:-4}; GS=${2:-"2 1"}; PS=${3:-"0/1 1/3 1/2 2/3 1/1"}
mkdir -p gpurun_out/pull
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for g in $GS; do for pl in $PS; do tag=n${N}_g${g}_p${pl/\//_}
$R --nproc-per-node $N --master-port 29$((RANDOM%800+100)) bench.py --gpus $N --steps 10 --warmup 3 --no-e2e --no-comparators --groups $g --intra-pull $pl > gpurun_out/pull/$tag.json 2> gpurun_out/pull/$tag.err
python -c "
import json; d=json.loads(open('gpurun_out/pull/$tag.json').read().splitlines()[-1]); k=d['kernels']; print('$tag', d['config']['M'],'x',d['config']['N'], d['ms_per_step'], {n[:2]: v['avg_ms'] for n,v in k.items()}, 'tlq', d['collectives']['tlq_hs_reduce_scatter']['ms'])" || tail -3 gpurun_out/pull/$tag.err
done; done
