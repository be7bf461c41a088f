mkdir -p gpurun_out
./tools/dp_lat_bin; ./tools/dp_lat_prec_bin
bash tools/fp_profile.sh 2>&1 | tail -3
bash tools/fp_profile.sh -DSKYRX_FP_NO_TRAIL 2>&1 | tail -3
