set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 300 python tools/prof_step.py --config 1 --steps 2 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg1.csv python tools/prof_step.py --config 1 --steps 2 > gpurun_out/ncu1.log 2>&1 ; \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_build_tc -s 1 -c 1 -o gpurun_out/prof_build python tools/prof_step.py --config 1 --steps 2 > gpurun_out/ncu2.log 2>&1
echo done
