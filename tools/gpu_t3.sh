# wide finalize (finalize_wide.cu) + vectorised tcw_pack: tests, latency, c3 bench + launch list
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_finalize.py -q -x -p no:randomly 2>&1 | tail -15
BANDS=128,270 timeout 300 python tools/time_finalize.py 2>&1 | tail -12
timeout 900 python -m pytest tests/test_gpu_geometry.py -k c3 tests/test_gpu_parity.py -k "wide" -q -x -p no:randomly 2>&1 | tail -5
timeout 600 python bench.py --config c3 --no-cpu --no-e2e > gpurun_out/t3_c3.log 2>&1; echo "c3 rc=$?"; tail -1 gpurun_out/t3_c3.log | cut -c1-400
C3="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --no-graph"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t3_launches_c3.csv $C3 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/t3_launches_c3.csv | head -14
