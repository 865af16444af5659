# prep kernels after the k_norms change: GPU tests, a headline bench line, ncu of k_norms
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t29.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/t29.log
timeout 900 python bench.py --extra "1,3" --no-cpu-baseline > gpurun_out/b29.json 2> gpurun_out/b29.err; echo "bench $?"
python tools/summ.py gpurun_out/b29.json 2>/dev/null | head -10
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum -k regex:k_norms -c 2 python tools/prof_step.py --config 4 --steps 1 2>&1 | grep -E "k_norms|duration|bytes_read" | head -8
