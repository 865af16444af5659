# Round-2 GPU evidence (one gpurun call; every ncu capture after the same command ran clean):
#   launch list of the headline bench step (cfg4), ncu --set full of the hot kernels.
mkdir -p gpurun_out
set -x
timeout 600 python bench.py --extra "" --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --parity-users 16 > gpurun_out/p_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg4.csv \
  python bench.py --extra "" --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --parity-users 16 > gpurun_out/p_ncu_ll.log 2>&1
echo "launch list rc=$?"
timeout 300 python tools/prof_step.py --config 4 --steps 1 > gpurun_out/p4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_query_tc|k_exact_select|k_exact_decide|k_bits_emit" -s 4 -c 5 -o gpurun_out/r02_cfg4_query -f \
  python tools/prof_step.py --config 4 --steps 1 > gpurun_out/p_ncu4.log 2>&1
echo "cfg4 query rc=$?"
timeout 300 python tools/prof_step.py --config 4 --n 37888 --steps 1 > gpurun_out/p4b.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_build_tc2cta" -c 1 -o gpurun_out/r02_cfg4_build -f \
  python tools/prof_step.py --config 4 --n 37888 --steps 1 > gpurun_out/p_ncu4b.log 2>&1
echo "cfg4 build rc=$?"
timeout 300 python tools/prof_step.py --config 3 --steps 1 > gpurun_out/p3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_query_tc|k_build_tc|k_exact_select" -s 1 -c 3 -o gpurun_out/r02_cfg3 -f \
  python tools/prof_step.py --config 3 --steps 1 > gpurun_out/p_ncu3.log 2>&1
echo "cfg3 rc=$?"
timeout 300 python tools/prof_step.py --config 3 --steps 1 --pprime 2 > gpurun_out/p3p.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_verify_scan" -s 1 -c 1 -o gpurun_out/r02_cfg3_scan -f \
  python tools/prof_step.py --config 3 --steps 1 --pprime 2 > gpurun_out/p_ncu3p.log 2>&1
echo "cfg3 scan rc=$?"
timeout 300 python tools/prof_step.py --config 1 --steps 2 > gpurun_out/p1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_build_tc|k_exact_select|k_query_tc" -s 3 -c 3 -o gpurun_out/r02_cfg1 -f \
  python tools/prof_step.py --config 1 --steps 2 > gpurun_out/p_ncu1.log 2>&1
echo "cfg1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_norms|k_prep_users|k_prep_items" -c 3 -o gpurun_out/r02_cfg4_prep -f \
  python tools/prof_step.py --config 4 --steps 1 > gpurun_out/p_ncu4p.log 2>&1
echo "cfg4 prep rc=$?"
