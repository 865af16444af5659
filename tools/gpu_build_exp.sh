# Build-contraction experiments on the cfg4 shape (dev library switches, tools/time_build.py).
mkdir -p gpurun_out
export RMIPS_LIB=$PWD/paper_2110_07131_b200/librmips_dev.so
N=${N:-37888}
timeout 600 python tools/time_build.py $N 1000000 200 50 3 RMIPS_NO_2CTA=1 default RMIPS_NO_2CTA=1 default
