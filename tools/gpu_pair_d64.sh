# d <= 64: CTA-pair kernel (now with its seed pass) vs k_build_tc on configs[1..3]
mkdir -p gpurun_out
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
for c in cfg1 cfg2 cfg3; do timeout 400 python tools/time_build.py $c 0 0 0 5 default RMIPS_2CTA_D64=1 default RMIPS_2CTA_D64=1; done > gpurun_out/pair_d64.log 2>&1
cat gpurun_out/pair_d64.log
