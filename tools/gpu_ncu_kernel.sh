# ncu --set full capture of one launch of kernel regex $1 (second step of tools/prof_step.py, cfg $2)
mkdir -p gpurun_out
K=$1; CFG=${2:-1}
timeout 300 python tools/prof_step.py --config $CFG --steps 2 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" -s 1 -c 1 -o gpurun_out/prof_k -f python tools/prof_step.py --config $CFG --steps 2 > gpurun_out/ncu_k.log 2>&1
echo "ncu rc=$?"
