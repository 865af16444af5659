# ncu --set full (source sampling) of the regrouped configs[4] build's MAIN pass (second build, launch 4)
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:k_build_tc2cta" -s 3 -c 1 -o gpurun_out/main_pass -f python tools/build_once.py 4 > gpurun_out/ncu_main.log 2>&1
echo "ncu rc=$?"
