# Same-box A/B of the exact select (B5): librmips_selbase.so (committed) vs librmips_dev.so / _sel1.so
# (working tree, 2 or 1 CTAs per SM); build - contraction = prep + select + blocks
for L in selbase dev sel1 selbase dev sel1; do
  RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_$L.so timeout 300 python tools/time_build.py 296000 1000000 200 50 3 default | sed "s/^/$L /"
done > gpurun_out/sel_ab.log 2>&1
for c in cfg1 cfg3; do for L in selbase dev sel1; do
  RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_$L.so timeout 300 python tools/time_build.py $c 0 0 0 5 default | sed "s/^/$L /"
done; done >> gpurun_out/sel_ab.log 2>&1
cat gpurun_out/sel_ab.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t27.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/t27.log
