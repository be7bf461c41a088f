cd "$(dirname "$0")/.."
python tools/stage_probe.py 2>&1 | tail -12
python tools/air_kernels_case.py > gpurun_out/air_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_air.csv python tools/air_kernels_case.py > /dev/null 2>&1
echo rc=$?
