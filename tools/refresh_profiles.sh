# One-GPU profile refresh: the bench line, the ncu launch list of the same command and one
# `ncu --set full` capture of K1..K5 (each only after the plain command exited 0).
set -e
mkdir -p gpurun_out/prof
python bench.py --steps 10 --warmup 3 > gpurun_out/prof/bench_n1.json 2> gpurun_out/prof/bench_n1.err
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k[1-5]_" -c 5 -o gpurun_out/prof/full \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-comparators > gpurun_out/prof/ncu_full.log 2>&1
echo done
