mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -k "raw_byte_moments or wide" tests/test_gpu_geometry.py::test_c3_full_cube -q -p no:randomly -x 2>&1 | tail -2
C3="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --no-graph"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/s13_launches_c3.csv $C3 > /dev/null 2>&1; echo "ncu rc=$?"
grep -E "raww_gram|Grid" gpurun_out/s13_launches_c3.csv | awk -F'","' '{print $13, $15}'
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"raww_gram_kernel" -c 1 -o gpurun_out/s13_raww -f $C3 > /dev/null 2>&1; echo "ncu full rc=$?"
timeout 300 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/s13_c3.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/s13_c3.json'));print('c3', d['value']/1e9, d['ms_per_step'], d['roofline']['frac'], d['roofline']['other_pass'], d.get('parity',{}).get('pass'))"
