# append-threshold fold (candq.cuh): parity tests of the 4-byte-list kernels, cfg4 build timing, head-pass launch times
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "regroup or cfg4 or cta_pair or trimmed or large_d or kmax_128 or above_2pow20 or random_instances" > gpurun_out/candq_tests.log 2>&1; echo "rc=$?" >> gpurun_out/candq_tests.log
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
timeout 900 python tools/time_build.py cfg4 0 0 0 5 RMIPS_HEAD_TILES=32 RMIPS_HEAD_TILES=0 > gpurun_out/candq_ab.log 2>&1
RMIPS_HEAD_TILES=32 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_build|k_gather" --log-file gpurun_out/candq_launch.csv python tools/build_once.py 4 > gpurun_out/candq_ncu.log 2>&1
cat gpurun_out/candq_ab.log
