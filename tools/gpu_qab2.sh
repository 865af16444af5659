# Same-box A/B of the query path: librmips_qbase.so (committed) vs librmips_dev.so (working tree); GPU tests
for c in 4 3 1; do
  for L in qbase dev qbase dev; do
    RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_$L.so timeout 300 python tools/time_query.py $c 2 default | sed "s/^/$L /"
  done
done > gpurun_out/qab2.log 2>&1
cat gpurun_out/qab2.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t32.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/t32.log
