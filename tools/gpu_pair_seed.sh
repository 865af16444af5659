# CTA-pair seed pass: parity tests, configs[4] A/B (seed on / off), head/main launch times
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "seed or regroup or cfg4 or cta_pair or trimmed or large_d or kmax_128 or above_2pow20 or random_instances or cfg0" > gpurun_out/pseed_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pseed_tests.log
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
timeout 900 python tools/time_build.py cfg4 0 0 0 3 RMIPS_SEED_TILES=8 RMIPS_SEED_TILES=0 RMIPS_SEED_TILES=8 RMIPS_SEED_TILES=0 > gpurun_out/pseed_ab.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_build|k_gather" --log-file gpurun_out/pseed_launch.csv python tools/build_once.py 4 > gpurun_out/pseed_ncu.log 2>&1
cat gpurun_out/pseed_ab.log
