cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python tools/time_calbin.py build/bin2/libskyrx_b200.so
python tools/time_calbin.py
for lib in build/bin2/libskyrx_b200.so paper_2602_13509_b200/libskyrx_b200.so; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:calibrate_bin -c 3 python tools/time_calbin.py $lib 2>&1 | grep -E "calibrate_bin_tiled|duration|bytes" | head -8
done
