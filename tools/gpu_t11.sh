cd "$(dirname "$0")/.."
C3="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --no-graph"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t11_c3.csv $C3 > /dev/null 2>&1; echo rc=$?
python tools/launch_summary.py gpurun_out/t11_c3.csv 2>/dev/null | head -5
