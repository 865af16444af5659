# d <= 64 CTA-pair kernel with 8-byte lists (FPol): parity + A/B against k_build_tc on configs[1..3]
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "d64 or regroup or cta_pair or seed" > gpurun_out/fpol_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fpol_tests.log
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
for c in cfg1 cfg2 cfg3; do timeout 400 python tools/time_build.py $c 0 0 0 5 default RMIPS_2CTA_D64=1,RMIPS_2CTA_FPOL=1 RMIPS_2CTA_D64=1,RMIPS_2CTA_FPOL=2 default RMIPS_2CTA_D64=1,RMIPS_2CTA_FPOL=2; done > gpurun_out/fpol_ab.log 2>&1
cat gpurun_out/fpol_ab.log
