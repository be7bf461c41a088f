mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_finalize.py -q -p no:randomly -x > gpurun_out/s2_fin.log 2>&1; echo "fin tests rc=$?"; tail -15 gpurun_out/s2_fin.log
timeout 300 python tools/time_finalize.py > gpurun_out/s2_time_fin.log 2>&1; echo "time rc=$?"; cat gpurun_out/s2_time_fin.log
timeout 300 python tools/debug_air_depth.py > gpurun_out/s2_air.log 2>&1; echo "air rc=$?"; tail -20 gpurun_out/s2_air.log
C3="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --no-graph"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"raww_gram_kernel" -c 1 -o gpurun_out/s2_raww -f $C3 > gpurun_out/s2_ncu_raww.log 2>&1; echo "ncu rc=$?"
