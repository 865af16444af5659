# Development A/B of the d <= 64 build (k_build_tc) on configs[1..3] (librmips_dev.so switches).
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
for c in cfg1 cfg2 cfg3; do timeout 300 python tools/time_build.py $c 0 0 0 5 default RMIPS_FLAT_SLOW=1 RMIPS_SEED_TILES=8 RMIPS_SLOW_LIMIT=16; done > gpurun_out/tb18.log 2>&1
cat gpurun_out/tb18.log
unset RMIPS_LIB
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t18.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/t18.log
