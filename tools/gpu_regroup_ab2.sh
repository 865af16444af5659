# Regrouped builds: tests (d = 50 and 100), d <= 64 A/B on configs[1..3], launch lists of the cfg4 build passes.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "regroup or cfg3 or cfg1_full" > gpurun_out/regroup_tests2.log 2>&1; echo "rc=$?" >> gpurun_out/regroup_tests2.log
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
for c in cfg3 cfg2 cfg1; do timeout 300 python tools/time_build.py $c 0 0 0 5 RMIPS_HEAD_TILES=0 RMIPS_HEAD_TILES=8 RMIPS_HEAD_TILES=16 RMIPS_HEAD_TILES=0 RMIPS_HEAD_TILES=8; done > gpurun_out/regroup_ab_d50.log 2>&1
for h in 16 32; do
RMIPS_HEAD_TILES=$h timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_build|k_gather|Onesweep|k_iota" --log-file gpurun_out/regroup_launch_h$h.csv python tools/build_once.py 4 > gpurun_out/regroup_ncu_h$h.log 2>&1
done
cat gpurun_out/regroup_ab_d50.log
