# ncu --set full (source sampling) of the regrouped build's head pass on configs[4]; head-length A/B
mkdir -p gpurun_out
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
timeout 900 python tools/time_build.py cfg4 0 0 0 3 RMIPS_HEAD_TILES=24 RMIPS_HEAD_TILES=32 RMIPS_HEAD_TILES=40 RMIPS_HEAD_TILES=24 RMIPS_HEAD_TILES=32 RMIPS_HEAD_TILES=40 > gpurun_out/head_ab.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_build_tc2cta" -s 2 -c 1 -o gpurun_out/head_pass -f python tools/build_once.py 4 > gpurun_out/ncu_head.log 2>&1
echo "ncu rc=$?"
cat gpurun_out/head_ab.log
