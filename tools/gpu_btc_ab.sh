# Same-box A/B of the d <= 64 build: librmips_btcbase.so (committed) vs librmips_dev.so (working tree)
for c in cfg1 cfg2 cfg3; do for L in btcbase dev btcbase dev; do
  RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_$L.so timeout 300 python tools/time_build.py $c 0 0 0 5 default | sed "s/^/$L /"
done; done > gpurun_out/btc_ab.log 2>&1
cat gpurun_out/btc_ab.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t35.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/t35.log
