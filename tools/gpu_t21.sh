cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream.py tests/test_gpu_strips.py -q -p no:randomly -k "clamp or stream or Stream or strips or Strip or raw_byte" 2>&1 | tail -1
python tools/time_cliff.py 2>&1 | tail -4
timeout 600 python bench.py --config c2 --no-cpu > gpurun_out/t21_c2.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/t21_c2.json').read().strip().splitlines()[-1]); print('c2', d['ms_per_step'], d['latency_ms_per_chunk']['device_resident'])"
