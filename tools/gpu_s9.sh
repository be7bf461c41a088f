mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_finalize.py -q -p no:randomly -x 2>&1 | tail -15
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s9_launches_fin.csv python tools/time_finalize.py > gpurun_out/s9_time_fin.log 2>&1; echo "ncu fin rc=$?"
python tools/launch_summary.py gpurun_out/s9_launches_fin.csv | head -14
timeout 300 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/s9_c3.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/s9_c3.json'));print('c3', d['value']/1e9, d['ms_per_step'], d['roofline']['frac'], d.get('parity'))"
