# Query filter A/B (librmips_dev.so switches); then the GPU tests
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
for c in 4 3 1; do timeout 300 python tools/time_query.py $c 2 default RMIPS_Q_NO_SLOW=1 RMIPS_Q_EPI_SKIP=1; done > gpurun_out/qab.log 2>&1
cat gpurun_out/qab.log
unset RMIPS_LIB
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t24.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/t24.log
