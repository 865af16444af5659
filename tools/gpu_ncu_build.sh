# ncu --set full capture of one build-contraction launch (cfg given as $1, default 1)
mkdir -p gpurun_out
CFG=${1:-1}
timeout 300 python tools/prof_step.py --config $CFG --steps 2 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_build_tc -s 1 -c 1 -o gpurun_out/prof_build_cfg$CFG -f python tools/prof_step.py --config $CFG --steps 2 > gpurun_out/ncu_build.log 2>&1
echo "ncu rc=$?"
