# single-launch query prep: GPU tests of the query paths + per-call timing A/B (dev switch RMIPS_QPREP2)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/qprep_tests.log 2>&1; echo "rc=$?" >> gpurun_out/qprep_tests.log
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
timeout 600 python tools/time_query.py 4 5 default RMIPS_QPREP2=1 default RMIPS_QPREP2=1 > gpurun_out/qprep_tq4.log 2>&1
timeout 600 python tools/time_query.py 1 5 default RMIPS_QPREP2=1 default RMIPS_QPREP2=1 > gpurun_out/qprep_tq1.log 2>&1
cat gpurun_out/qprep_tq4.log gpurun_out/qprep_tq1.log
