python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/dist2.log 2>&1; tail -3 gpurun_out/dist2.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
$TR bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-comparators > gpurun_out/b2_kernel.json 2> gpurun_out/b2_kernel.err
SDP4_WAIT_TIMEOUT_S=0 $TR bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-comparators > gpurun_out/b2_memop.json 2> gpurun_out/b2_memop.err
python -c "
import json
for f in ('b2_kernel','b2_memop'):
    d=json.load(open('gpurun_out/'+f+'.json')); print(f, d['ms_per_step'], d['collectives']['qwd_all_gather']['ms'], d['collectives']['tlq_hs_reduce_scatter']['ms'], d['comm_ops'])
"
