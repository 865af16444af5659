mkdir -p gpurun_out
timeout 600 python tools/prof_step.py --config 4 --n 37888 --steps 1 > gpurun_out/plain4.log 2>&1; echo plain rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_build_tcq -c 1 -o gpurun_out/prof_cfg4 -f python tools/prof_step.py --config 4 --n 37888 --steps 1 > gpurun_out/ncu4.log 2>&1; echo ncu rc=$?
