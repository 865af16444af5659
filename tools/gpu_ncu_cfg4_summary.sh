# ncu --set full of the cfg4-shaped build kernel (k_build_tcq, d = 200, m = 1M; n reduced to 2 user
# tiles per SM so the capture stays short) and of the P' verification scan (cfg1, --pprime 2).
mkdir -p gpurun_out
timeout 600 python tools/prof_step.py --config 4 --n 37888 --steps 1 > gpurun_out/plain4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_build_tcq -c 1 -o gpurun_out/prof_cfg4 -f \
  python tools/prof_step.py --config 4 --n 37888 --steps 1 > gpurun_out/ncu4.log 2>&1; echo "ncu4 rc=$?"
