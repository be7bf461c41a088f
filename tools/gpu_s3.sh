mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_finalize.py tests/test_gpu_parity.py tests/test_gpu_geometry.py::test_c3_full_cube tests/test_gpu_reference_suite.py -q -p no:randomly > gpurun_out/s3_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/s3_tests.log | tail -15
timeout 300 python tools/time_finalize.py > gpurun_out/s3_time_fin.log 2>&1; echo "time rc=$?"; cat gpurun_out/s3_time_fin.log
for pace in 16 0 8 32; do
  SKYRX_RAWW_PACE=$pace timeout 300 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/s3_c3_p$pace.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/s3_c3_p$pace.json'));print('pace $pace', d['ms_per_step'], d['roofline']['other_pass'])"
done
C3="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --no-graph"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"raww_gram_kernel" -c 1 -o gpurun_out/s3_raww -f $C3 > gpurun_out/s3_ncu_raww.log 2>&1; echo "ncu rc=$?"
