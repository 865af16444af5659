# ncu --set full (source-level sampling) of k_build_tc on configs[1], sparse vs branch-free slow path
mkdir -p gpurun_out
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
timeout 300 python tools/prof_step.py --config 1 --steps 2 > gpurun_out/plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_build_tc" -s 1 -c 1 -o gpurun_out/btc_new -f python tools/prof_step.py --config 1 --steps 2 > gpurun_out/ncu_new.log 2>&1
echo "new rc=$?"
RMIPS_FLAT_SLOW=1 timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_build_tc" -s 1 -c 1 -o gpurun_out/btc_flat -f python tools/prof_step.py --config 1 --steps 2 > gpurun_out/ncu_flat.log 2>&1
echo "flat rc=$?"
