cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 120 tools/mma_rate_probe_bin 2>&1 | tee gpurun_out/t2_mma_rate.txt
C3="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --no-graph"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t2_launches_c3.csv $C3 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/t2_launches_c3.csv | head -30
