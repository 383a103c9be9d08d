python -m pytest tests/test_gpu_parity.py -x -q -k "qwd or qw" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for tpb in 0 1 2 4 8 16; do SDP4_K1_TPB=$tpb python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-comparators 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('tpb $tpb', d['ms_per_step'], {n:(v['avg_ms'],v['gbs']) for n,v in k.items()})"; done
