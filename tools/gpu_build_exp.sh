# Build-contraction experiments on the cfg4 shape (dev library switches, tools/time_build.py).
mkdir -p gpurun_out
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
N=${N:-37888}
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 500 > gpurun_out/exp_clocks.csv &
SMI=$!
for cfg in "default" "RMIPS_NO_CS=1" "RMIPS_EPI_SKIP=1" "RMIPS_EPI_SKIP=1 RMIPS_NOFEED=1" "RMIPS_NO_CS=1 RMIPS_NOFEED=1"; do
  env $cfg TAG="$cfg" timeout 300 python tools/time_build.py $N 1000000 200 50 3
done
kill $SMI
