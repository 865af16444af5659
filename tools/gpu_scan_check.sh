# last-CTA chunk scan in registers: full GPU tests + query timing (configs[4], [3])
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/scan_tests.log 2>&1; echo "rc=$?" >> gpurun_out/scan_tests.log
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
timeout 600 python tools/time_query.py 4 5 > gpurun_out/scan_tq4.log 2>&1
timeout 600 python tools/time_query.py 3 5 > gpurun_out/scan_tq3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_bits" --log-file gpurun_out/scan_launch.csv python tools/time_query.py 4 1 > gpurun_out/scan_ncu.log 2>&1
cat gpurun_out/scan_tq4.log gpurun_out/scan_tq3.log
