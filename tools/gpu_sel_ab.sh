# Timing of the exact select (B5) at the configs[4] shape and configs[1,3] (build - contraction)
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
timeout 300 python tools/time_build.py 296000 1000000 200 50 3 default > gpurun_out/sel_ab.log 2>&1
for c in cfg1 cfg3; do timeout 300 python tools/time_build.py $c 0 0 0 5 default; done >> gpurun_out/sel_ab.log 2>&1
cat gpurun_out/sel_ab.log
unset RMIPS_LIB
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t20.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/t20.log
