mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -k "raw_byte_moments or wide" tests/test_gpu_geometry.py::test_c3_full_cube -q -p no:randomly > gpurun_out/s1_c3tests.log 2>&1; echo "c3 tests rc=$?"; tail -3 gpurun_out/s1_c3tests.log
C3="python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity"
timeout 300 $C3 > gpurun_out/s1_c3.json 2> gpurun_out/s1_c3.err; echo "c3 bench rc=$?"; tail -c 1500 gpurun_out/s1_c3.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s1_launches_c3.csv python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --no-graph > /dev/null 2>&1; echo "ncu rc=$?"
timeout 300 python tools/debug_air_depth.py > gpurun_out/s1_air.log 2>&1; echo "air rc=$?"; cat gpurun_out/s1_air.log | tail -20
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_strips.py -q -p no:randomly > gpurun_out/s1_rest.log 2>&1; echo "rest rc=$?"; tail -3 gpurun_out/s1_rest.log
