# A/B of development library variants (paper_2110_07131_b200/librmips_<v>.so, built with
# build_lib.build(variant=...)) and env switches: cfg1 and cfg3 bench lines per variant.
# Usage: gpu_ab.sh v1 v2:ENV=1 ...   ("base" = librmips.so; CFGS="1 3" overrides the configs)
mkdir -p gpurun_out
for spec in "$@"; do
  v=${spec%%:*}; envs=""; [ "$spec" != "$v" ] && envs=${spec#*:}
  lib=paper_2110_07131_b200/librmips_$v.so; [ "$v" = base ] && lib=paper_2110_07131_b200/librmips.so
  for c in ${CFGS:-1 3}; do
    tag=$(echo "${spec}_cfg$c" | tr ':=,' '___')
    env $envs RMIPS_LIB=$PWD/$lib timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
    python -c "
import json; d=json.load(open('gpurun_out/ab_$tag.json')); b=d['build']; q=d['query']
print('%-28s cfg$c step %.3f contraction %.3f select %.3f cand/u %.1f query %.3f' % ('$spec', d['ms_per_step'], b['contraction_ms'], b['select_blocks_ms'], b['candidates_per_user'], q['ms']))"
  done
done
