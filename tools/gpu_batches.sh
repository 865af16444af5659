# batched query API: GPU tests, then the headline bench with both query APIs (same box)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t28.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/t28.log
timeout 900 python bench.py --extra "" > gpurun_out/b28_batches.json 2> gpurun_out/b28_batches.err; echo "bench batches $?"
timeout 900 python bench.py --extra "" --query-api calls --no-cpu-baseline > gpurun_out/b28_calls.json 2> gpurun_out/b28_calls.err; echo "bench calls $?"
for f in b28_batches b28_calls; do echo $f; python tools/summ.py gpurun_out/$f.json 2>/dev/null | head -7; done
tail -3 gpurun_out/b28_batches.err
