mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -k "TestFastMode" -q -p no:randomly 2>&1 | tail -2
PYTHONPATH=. python tools/stage_probe.py 2>&1 | tail -10
for c in "" --dead --gains; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s18_cliff$c.csv python tools/cliff_case.py $c > /dev/null 2>&1; echo "ncu $c rc=$?"
python tools/launch_summary.py gpurun_out/s18_cliff$c.csv | head -12
done
