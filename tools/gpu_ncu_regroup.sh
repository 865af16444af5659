# ncu metrics of the regrouped configs[4] build at full size: head pass and main pass (second build)
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__cycles_elapsed.avg
timeout 1500 ncu --metrics $M --clock-control none --csv -k regex:"k_build_tc2cta" -s 2 -c 2 --log-file gpurun_out/regroup_metrics.csv python tools/build_once.py 4 > gpurun_out/regroup_metrics.log 2>&1
echo "ncu rc=$?"
