cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_finalize.py -q -x -p no:randomly 2>&1 | tail -4
BANDS=270 timeout 300 python tools/time_finalize.py 2>&1 | tail -4
bash tools/fw_profile.sh 2>&1 | tail -1
