cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in "" --dead --gains; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t7_cliff$c.csv python tools/cliff_case.py $c > /dev/null 2>&1; echo "ncu $c rc=$?"
python tools/launch_summary.py gpurun_out/t7_cliff$c.csv 2>/dev/null | head -14
done
