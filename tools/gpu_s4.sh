mkdir -p gpurun_out
timeout 300 python bench.py --no-e2e --no-cpu > gpurun_out/s4_c4.json 2> gpurun_out/s4_c4.err; echo "c4 rc=$?"
python -c "import json;d=json.load(open('gpurun_out/s4_c4.json'));print('c4', d['value']/1e9, d['ms_per_step'], d['roofline']['frac'], d['roofline']['other_pass'], d['clocks'], d.get('parity',{}).get('pass'))"
timeout 300 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/s4_c3.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/s4_c3.json'));print('c3', d['value']/1e9, d['ms_per_step'], d['roofline'])"
timeout 300 python bench.py --config c5 --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/s4_c5.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/s4_c5.json'));print('c5', d['value']/1e9, d['ms_per_step'], d['roofline'])"
C4="python bench.py --strips 1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --no-graph"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4_launches_c4.csv $C4 > /dev/null 2>&1; echo "ncu c4 rc=$?"
C3="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --no-graph"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4_launches_c3.csv $C3 > /dev/null 2>&1; echo "ncu c3 rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4_launches_fin.csv python tools/time_finalize.py > /dev/null 2>&1; echo "ncu fin rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/s4_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/s4_pytest.log | tail -12
