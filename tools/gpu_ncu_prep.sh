# ncu of the build prep kernels (configs[4] size): duration, DRAM bytes, throughput
mkdir -p gpurun_out
timeout 300 python tools/prof_step.py --config 4 --steps 1 > gpurun_out/plain_prep.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_norms|k_prep_users|k_prep_items|k_split_sorted|Onesweep|k_blocks" -c 12 -o gpurun_out/prep4 -f python tools/prof_step.py --config 4 --steps 1 > gpurun_out/ncu_prep.log 2>&1
echo "prep rc=$?"
