# d <= 64 regroup with saved head state: parity (forced on), A/B of the head length on configs[3], [2], [1]
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "regroup or cfg3 or variants" > gpurun_out/probe3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/probe3_tests.log
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
for c in cfg3 cfg2 cfg1; do timeout 400 python tools/time_build.py $c 0 0 0 5 RMIPS_HEAD_TILES=0 RMIPS_HEAD_TILES=8 RMIPS_HEAD_TILES=4 RMIPS_HEAD_TILES=12 RMIPS_HEAD_TILES=0 RMIPS_HEAD_TILES=8; done > gpurun_out/probe3_ab.log 2>&1
RMIPS_HEAD_TILES=8 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_build|k_gather" --log-file gpurun_out/probe3_cfg3_h8.csv python tools/build_once.py 3 > gpurun_out/probe3_ncu.log 2>&1
cat gpurun_out/probe3_ab.log
