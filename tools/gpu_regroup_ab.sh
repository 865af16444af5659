# Regrouped CTA-pair build: parity tests, then A/B of the head-pass length on the configs[4] shape.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "regroup or cfg4 or cta_pair or trimmed" > gpurun_out/regroup_tests.log 2>&1; echo "rc=$?" >> gpurun_out/regroup_tests.log
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
timeout 900 python tools/time_build.py cfg4 0 0 0 3 RMIPS_HEAD_TILES=0 RMIPS_HEAD_TILES=32 RMIPS_HEAD_TILES=16 RMIPS_HEAD_TILES=48 RMIPS_HEAD_TILES=0 RMIPS_HEAD_TILES=32 > gpurun_out/regroup_ab.log 2>&1
cat gpurun_out/regroup_ab.log
