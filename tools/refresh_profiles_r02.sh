# One-GPU evidence for profiles/r02: the driver's bench command, the ncu launch list of exactly
# the warm-up + timed steps (--steps-only), and one `ncu --set full` capture of K1 and the fused
# world-1 TLq-HS kernel (K345) of the same workload (each ncu only after its plain command
# exited 0).  K3 / K4 / K5 alone (what each rank of a P > 1 job runs) are timed by bench.py's
# three_kernel_tlq variant; THREE_KERNEL=1 captures them instead (sdp4 local fusion off).
mkdir -p gpurun_out/prof
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/prof/bench_n1.json 2> gpurun_out/prof/bench_n1.err
python bench.py --steps 20 --warmup 5 --steps-only > gpurun_out/prof/so.json 2>/dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_steps_only.csv \
    python bench.py --steps 20 --warmup 5 --steps-only > gpurun_out/prof/ncu_launch.log 2>&1
if [ -n "$THREE_KERNEL" ]; then
  SDP4_NO_LOCAL_FUSION=1 python bench.py --steps 3 --warmup 3 --steps-only > /dev/null 2>&1 && \
  SDP4_NO_LOCAL_FUSION=1 ncu --set full --clock-control none --import-source on -k regex:"k3_tlq|k4_tlq|k5_tlq" -s 9 -c 3 \
      -o gpurun_out/prof/full3 python bench.py --steps 3 --warmup 3 --steps-only > gpurun_out/prof/ncu_full3.log 2>&1
else
  python bench.py --steps 3 --warmup 3 --steps-only > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k1_qwd|k_tlq_local" -s 6 -c 2 \
      -o gpurun_out/prof/full python bench.py --steps 3 --warmup 3 --steps-only > gpurun_out/prof/ncu_full.log 2>&1
fi
echo done
