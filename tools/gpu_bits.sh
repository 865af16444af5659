# bit-matrix output with all 32 word loads of a block in flight: GPU tests, kernel times, bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/bits_tests.log 2>&1; echo "rc=$?" >> gpurun_out/bits_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_bits|k_lemma3|k_query_norms|k_query_finish" --log-file gpurun_out/bits_launch.csv python tools/time_query.py 4 1 > gpurun_out/bits_ncu.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
