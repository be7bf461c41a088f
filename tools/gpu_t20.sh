cd "$(dirname "$0")/.."
python tools/time_sc_ab.py tools/_var/gr_old/libskyrx_b200.so tools/_var/gr_new/libskyrx_b200.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream.py tests/test_gpu_geometry.py -q -p no:randomly -k "raw_byte or own_shift or clamp or stream or c4 or c2 or c5 or deterministic or c1_full" 2>&1 | tail -1
timeout 600 python bench.py --config c2 --no-cpu > gpurun_out/t20_c2.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/t20_c2.json').read().strip().splitlines()[-1]); print('c2', d['ms_per_step'], d['latency_ms_per_chunk'])"
timeout 600 python bench.py --config c1 --no-cpu > gpurun_out/t20_c1.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/t20_c1.json').read().strip().splitlines()[-1]); print('c1', d['value'], d['ms_per_step'])"
