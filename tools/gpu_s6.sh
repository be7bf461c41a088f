mkdir -p gpurun_out
bash tools/fp_profile.sh > gpurun_out/s6_fp.log 2>&1; tail -4 gpurun_out/s6_fp.log
timeout 600 python -m pytest tests/test_gpu_finalize.py -q -p no:randomly > gpurun_out/s6_fin.log 2>&1; echo "fin rc=$?"; tail -3 gpurun_out/s6_fin.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s6_launches_fin.csv python tools/time_finalize.py > /dev/null 2>&1; echo "ncu fin rc=$?"
python tools/launch_summary.py gpurun_out/s6_launches_fin.csv
timeout 300 python bench.py --no-e2e --no-cpu --no-parity > gpurun_out/s6_c4.json 2> gpurun_out/s6_c4.err; echo "c4 rc=$?"
python -c "import json;d=json.load(open('gpurun_out/s6_c4.json'));print('c4', d['value']/1e9, d['ms_per_step'], d['roofline']['frac'], d['roofline']['ms_per_launch'], d['roofline']['other_pass'], d['clocks'])"
