# bench lines for the parity configs 2-4 (evidence; the driver's bench line is configs[1])
mkdir -p gpurun_out
for c in 2 3 4; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err
  echo "cfg$c rc=$?"
done
