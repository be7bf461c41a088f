cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_geometry.py tests/test_gpu_parity.py -q -x -p no:randomly -k "c3 or wide or raw_byte or own_shift or clamp" 2>&1 | tail -3
C3="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --no-graph"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t10_c3.csv $C3 > /dev/null 2>&1; echo rc=$?
python tools/launch_summary.py gpurun_out/t10_c3.csv 2>/dev/null | head -8
timeout 600 python bench.py --config c3 --no-cpu --no-e2e > gpurun_out/t10_c3.log 2>&1; tail -1 gpurun_out/t10_c3.log | cut -c1-330
