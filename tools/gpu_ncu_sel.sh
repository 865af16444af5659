# ncu --set full of k_exact_select at the configs[4] shape (n reduced: the per-row work is the same)
mkdir -p gpurun_out
timeout 300 python tools/prof_step.py --config 4 --n 148000 --steps 1 > gpurun_out/plain_sel.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_exact_select" -c 1 -o gpurun_out/sel4 -f python tools/prof_step.py --config 4 --n 148000 --steps 1 > gpurun_out/ncu_sel.log 2>&1
echo "sel rc=$?"
