# fp32 Cauchy-Schwarz bound (no DMUL in the epilogue): GPU tests, build timing on configs[4], [3], [1], bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pns_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pns_tests.log
for c in cfg4 cfg3 cfg1; do timeout 600 python tools/time_build.py $c 0 0 0 5; done > gpurun_out/pns_tb.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/pns_tb.log
