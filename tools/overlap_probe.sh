R() { n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) "$@"; }
for ov in "" "--overlap"; do R 4 bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --no-comparators --no-variants $ov 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$ov', d['ms_per_step'], d['value'])"; done
python bench.py --steps 20 --warmup 5 --no-e2e --no-comparators --no-variants --no-cpu-baseline --overlap 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('n1 overlap', d['ms_per_step'], d['value'])"
