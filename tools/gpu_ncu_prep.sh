# ncu --set full of the build prep kernels and the query exact-decide kernels at the configs[4] size
mkdir -p gpurun_out
timeout 300 python tools/prof_step.py --config 4 --steps 1 > gpurun_out/plain_prep.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_norms|k_prep_users|k_prep_items" -c 4 -o gpurun_out/prep4 -f python tools/prof_step.py --config 4 --steps 1 > gpurun_out/ncu_prep.log 2>&1
echo "prep rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_scan_compact|k_exact_decide" -s 20 -c 4 -o gpurun_out/dec4 -f python tools/prof_step.py --config 4 --steps 1 > gpurun_out/ncu_dec.log 2>&1
echo "dec rc=$?"
