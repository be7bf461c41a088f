cd "$(dirname "$0")/.."
python tools/air_kernels_case.py > gpurun_out/air_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:calibrate_bin_tiled -c 1 -o gpurun_out/calib_full -f python tools/air_kernels_case.py > gpurun_out/calib_ncu.log 2>&1
echo rc=$?
