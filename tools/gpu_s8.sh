mkdir -p gpurun_out
bash tools/fp_profile.sh 2>&1 | tail -3
bash tools/fp_profile.sh -DSKYRX_FP_NO_TRAIL 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_finalize.py -q -p no:randomly 2>&1 | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s8_launches_fin.csv python tools/time_finalize.py > /dev/null 2>&1; echo "ncu fin rc=$?"
python tools/launch_summary.py gpurun_out/s8_launches_fin.csv | grep -i panel
