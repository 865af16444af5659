# stale-theta checkpoint refresh, theta-only (librmips_dev.so RMIPS_STALE_EVERY; 0 = off), alternating, cfg4 shape
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
timeout 900 python tools/time_build.py 296000 1000000 200 50 3 RMIPS_STALE_EVERY=0 RMIPS_STALE_EVERY=16 RMIPS_STALE_EVERY=8 RMIPS_STALE_EVERY=0 RMIPS_STALE_EVERY=16 RMIPS_STALE_EVERY=8 RMIPS_STALE_EVERY=4 > gpurun_out/stale_ab.log 2>&1
timeout 900 python tools/time_build.py 148000 1000000 300 50 3 RMIPS_STALE_EVERY=0 RMIPS_STALE_EVERY=16 RMIPS_STALE_EVERY=0 RMIPS_STALE_EVERY=16 >> gpurun_out/stale_ab.log 2>&1
cat gpurun_out/stale_ab.log
unset RMIPS_LIB
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t39.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/t39.log
