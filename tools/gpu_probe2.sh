# (a) cfg3 d <= 64 regroup (restart form) launch times; (b) stale-theta period A/B on the regrouped cfg4 build
mkdir -p gpurun_out
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
RMIPS_HEAD_TILES=8 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_build|k_gather" --log-file gpurun_out/probe_cfg3_h8.csv python tools/build_once.py 3 > gpurun_out/probe_cfg3.log 2>&1
RMIPS_HEAD_TILES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_build|k_gather" --log-file gpurun_out/probe_cfg3_h0.csv python tools/build_once.py 3 >> gpurun_out/probe_cfg3.log 2>&1
timeout 900 python tools/time_build.py cfg4 0 0 0 3 RMIPS_STALE_EVERY=16 RMIPS_STALE_EVERY=0 RMIPS_STALE_EVERY=8 RMIPS_STALE_EVERY=32 RMIPS_STALE_EVERY=16 > gpurun_out/probe_stale.log 2>&1
cat gpurun_out/probe_stale.log
