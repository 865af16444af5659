# round check + the headline step's launch list (ncu gpu__time_duration, after the same command ran clean)
mkdir -p gpurun_out
bash tools/gpu_round_check.sh
timeout 600 python bench.py --extra "" --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --parity-users 16 > gpurun_out/p_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg4.csv \
  python bench.py --extra "" --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --parity-users 16 > gpurun_out/p_ncu_ll.log 2>&1
echo "launch list rc=$?"
