# BASELINE.json configs[2..3] at 4 GPUs: GPT-13B (2x2) and the group-size sweep 64/128/256.
mkdir -p gpurun_out/cfg
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
summ() { python -c "import json,sys;d=json.loads(open('$1').read().splitlines()[-1]);c=d.get('comparators') or {};print(d['config']['workload'],'value',d['value'],'ms',d['ms_per_step'],'speedup',c.get('speedup_vs_unquantized'),'e2e',(d.get('e2e') or {}).get('value'),{n:v['avg_ms'] for n,v in d['kernels'].items()})" || tail -3 ${1%.json}.err; }
$R --master-port 29701 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/cfg/b_1.3B_g2.json 2> gpurun_out/cfg/b_1.3B_g2.err; summ gpurun_out/cfg/b_1.3B_g2.json
for G in 64 256; do $R --master-port 2971$((G/64)) bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --group $G --qwd-group $G > gpurun_out/cfg/b_1.3B_G$G.json 2> gpurun_out/cfg/b_1.3B_G$G.err; summ gpurun_out/cfg/b_1.3B_G$G.json; done
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True $R --master-port 29720 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e --no-comparators --model 13B > gpurun_out/cfg/b_13B_g2.json 2> gpurun_out/cfg/b_13B_g2.err; summ gpurun_out/cfg/b_13B_g2.json
