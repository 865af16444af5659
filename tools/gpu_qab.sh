# Query filter dev A/B (librmips_dev.so) on configs[3], [4], [1]; GPU tests; bench (configs[4], 1, 3)
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
for c in 3 4 1; do timeout 300 python tools/time_query.py $c 2 default RMIPS_Q_EPI_SKIP=1 RMIPS_Q_EPI_SKIP=1,RMIPS_Q_NOFEED=1 RMIPS_Q_NO_SLOW=1; done > gpurun_out/qab.log 2>&1
cat gpurun_out/qab.log
unset RMIPS_LIB
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t30.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/t30.log
timeout 900 python bench.py --extra "1,2,3" --no-cpu-baseline > gpurun_out/b30.json 2> gpurun_out/b30.err; echo "bench $?"
python tools/summ.py gpurun_out/b30.json 2>/dev/null | head -12
