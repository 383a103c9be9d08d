mkdir -p gpurun_out/multi
R() { n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) "$@"; }
R 4 tools/size_sweep.py --graphs --out gpurun_out/multi/size_sweep_n4_2x2.json > gpurun_out/multi/size_2x2.log 2>&1; tail -13 gpurun_out/multi/size_2x2.log
R 4 tools/size_sweep.py --graphs --groups 1 --out gpurun_out/multi/size_sweep_n4_1x4.json > gpurun_out/multi/size_1x4.log 2>&1; tail -2 gpurun_out/multi/size_1x4.log
R 4 tools/size_sweep.py --graphs --groups 4 --out gpurun_out/multi/size_sweep_n4_4x1.json > gpurun_out/multi/size_4x1.log 2>&1; tail -2 gpurun_out/multi/size_4x1.log
