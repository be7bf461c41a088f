mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -k "TestFastMode or fused" -q -p no:randomly -s 2>&1 | grep -E "PARITY|passed|failed|Error" | tail -12
python tools/stage_probe.py 2>&1 | tail -10
python tools/time_cliff.py 2>&1 | tail -5
