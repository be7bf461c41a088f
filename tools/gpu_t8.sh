cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:randomly -k "quantis or radiance_cube or Fast or fast or gains or line_gains" 2>&1 | tail -4
timeout 600 python tools/time_cliff.py 2>&1 | tail -4
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gram_tc -c 4 python tools/cliff_case.py --gains 2>&1 | grep -E "gram_tc|duration" | head -8
