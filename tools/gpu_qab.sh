# Query filter dev A/B (librmips_dev.so): MMA N split vs default, alternating, configs[4], [3], [1]
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
for c in 4 3 1; do timeout 300 python tools/time_query.py $c 2 default RMIPS_Q_SPLITN=1 default RMIPS_Q_SPLITN=1; done > gpurun_out/qab.log 2>&1
cat gpurun_out/qab.log
