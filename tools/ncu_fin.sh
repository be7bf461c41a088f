# ncu --set full (source counters) of finalize_small_kernel over 148 matrices at B = $1
cd "$(dirname "$0")/.."
python tools/fin_ncu_case.py ${1:-70} > gpurun_out/fin_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:finalize_small -s 1 -c 1 -o gpurun_out/fin_small -f python tools/fin_ncu_case.py ${1:-70} > gpurun_out/fin_ncu.log 2>&1
echo rc=$?
