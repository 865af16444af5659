# programmatic dependent launch on the query chain: GPU tests, smoke, bench A/B with the dev library
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pdl_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pdl_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/pdl_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/pdl_smoke.log
D=$PWD/paper_2110_07131_b200/librmips_dev.so
for v in on off on off; do
  if [ $v = off ]; then export RMIPS_NO_PDL=1; else unset RMIPS_NO_PDL; fi
  RMIPS_LIB=$D timeout 600 python bench.py --extra 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/pdl_bench_$v.json 2>/dev/null
  python -c "import json;b=json.loads(open('gpurun_out/pdl_bench_$v.json').read().strip().splitlines()[-1]);print('$v', b['ms_per_step'], b['query']['ms'], b['e2e']['ms_per_step'], b['configs']['cfg1']['ms_per_step'], b['configs']['cfg1']['query']['ms'])" >> gpurun_out/pdl_ab.log
done
unset RMIPS_NO_PDL
cat gpurun_out/pdl_ab.log
