# A/B of a dev switch on the full cfg4 bench (contraction time, clocks): A = default, B = env $1
mkdir -p gpurun_out
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
for r in 1 2; do
  for v in A B; do
    if [ $v = B ]; then E="$1"; else E="X=1"; fi
    env $E timeout 300 python bench.py --config ${CFG:-4} --extra "" --no-e2e --no-cpu-baseline --parity-users 64 --steps 10 > gpurun_out/ab_$v$r.json 2>/dev/null
    python - "$v$r" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab_%s.json" % sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "step %.1f ms build %.1f contraction %.1f frac %.3f clocks %s parity %s" % (d["ms_per_step"], d["build"]["ms"], d["roofline"]["kernel_ms"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["parity"]["disagreements"]))
PY
  done
done
