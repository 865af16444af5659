# stale-theta checkpoint refresh in the d <= 64 kernel (theta-only), alternating: configs[1..3]
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
for c in cfg3 cfg1 cfg2; do timeout 300 python tools/time_build.py $c 0 0 0 5 RMIPS_STALE_EVERY=0 RMIPS_STALE_EVERY=16 RMIPS_STALE_EVERY=0 RMIPS_STALE_EVERY=16 RMIPS_STALE_EVERY=32; done > gpurun_out/stale_ab.log 2>&1
cat gpurun_out/stale_ab.log
