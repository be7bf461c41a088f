# session-4: finalize phase profile + K3 timings + c2 per-kernel launch list
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/fp_profile.sh > gpurun_out/s4_fp_profile.txt 2>&1; tail -4 gpurun_out/s4_fp_profile.txt
BANDS=70 PYTHONPATH=. timeout 300 python tools/time_finalize.py > gpurun_out/s4_fin.txt 2>&1; cat gpurun_out/s4_fin.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4_launches_c2.csv python bench.py --config c2 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1; echo "ncu c2 rc=$?"
python tools/launch_summary.py gpurun_out/s4_launches_c2.csv 2>&1 | head -30
echo done
