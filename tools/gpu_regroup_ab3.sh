# Regrouped CTA-pair build with saved head state: tests, cfg4 A/B of the head length, launch list.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "regroup or cfg4 or cta_pair or trimmed or large_d or kmax_128 or above_2pow20" > gpurun_out/regroup_tests3.log 2>&1; echo "rc=$?" >> gpurun_out/regroup_tests3.log
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
timeout 900 python tools/time_build.py cfg4 0 0 0 3 RMIPS_HEAD_TILES=0 RMIPS_HEAD_TILES=32 RMIPS_HEAD_TILES=16 RMIPS_HEAD_TILES=48 RMIPS_HEAD_TILES=64 RMIPS_HEAD_TILES=0 RMIPS_HEAD_TILES=32 > gpurun_out/regroup_ab3.log 2>&1
RMIPS_HEAD_TILES=32 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_build|k_gather" --log-file gpurun_out/regroup3_launch_h32.csv python tools/build_once.py 4 > gpurun_out/regroup3_ncu.log 2>&1
cat gpurun_out/regroup_ab3.log
