cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests/test_gpu_strips.py tests/test_gpu_geometry.py tests/test_gpu_parity.py -q -p no:randomly -k "strips or Strip or c4 or topk or Topk or mask or detect_batch" 2>&1 | tail -1
for ov in 0 1 0 1; do SKYRX_B200_MASK_OVERLAP=$ov timeout 900 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/t25_c4_$ov.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/t25_c4_$ov.json').read().strip().splitlines()[-1]); r=d['roofline']; print('overlap=$ov', round(d['value']/1e9,3), round(d['ms_per_step'],2), round(r['frac'],3), round(r['other_pass']['frac'],3), d['clocks']['sm_mhz'], d['parity']['pass'], d.get('invalid'))"; done
