# Round profiling: full bench line, per-launch device times (ncu launch list, cold-cache and
# serialised), and one ncu --set full capture of each hot kernel.  Results under gpurun_out/;
# summaries are copied to profiles/ by tools/summarize_profiles.py.
mkdir -p gpurun_out
CFG=${CFG:-1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
timeout 300 python tools/prof_step.py --config $CFG --steps 2 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg$CFG.csv \
    python tools/prof_step.py --config $CFG --steps 2 > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:k_build_tc|k_query_tc|k_exact_select' \
    -s 3 -c 3 -o gpurun_out/prof_cfg$CFG -f python tools/prof_step.py --config $CFG --steps 2 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
