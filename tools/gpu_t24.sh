cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_geometry.py tests/test_gpu_strips.py -q -p no:randomly -k "topk or Topk or mask or tensor_core_score or exact_digit or wide or c4 or c3 or c5 or c1 or strips or Strip or detect" 2>&1 | tail -1
timeout 900 python bench.py --no-cpu > gpurun_out/t24_c4.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/t24_c4.json').read().strip().splitlines()[-1]); r=d['roofline']; print('c4', d['value'], d['ms_per_step'], r['frac'], r['ms_per_launch'], r['other_pass']['frac'], d['hbm_fraction_whole_path'], d['clocks'], d['parity']['pass'])"
