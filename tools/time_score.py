"""Time the score and moments kernels alone on one c4 strip (CUDA events)."""
import os, sys, json
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2602_13509_b200 as P
from paper_2602_13509_b200.synth import Scene

L, S, B = 16384, 900, 70
sc = Scene(4000, S, B, 5)
raw = sc.generate(0, L)
d, c = torch.from_numpy(sc.dark).cuda(), torch.from_numpy(sc.coeff).cuda()
g = torch.ones(L, dtype=torch.float32, device='cuda')
plan = P.DetectPlan(L, S, B)
plan.run(0, raw, d, c, g, gain_const=1.0).finalize().score(0, raw, d, c, g)
torch.cuda.synchronize()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
res = {'stats_ms': t(lambda: plan.run(0, raw, d, c, g, gain_const=1.0)),
       'select_ms': t(lambda: plan.score(0, raw, d, c, g)) - t(lambda: plan.score_only(0, raw, d, c, g, topk_hist0=True)),
       'score_path_ms': t(lambda: plan.score(0, raw, d, c, g))}
print(json.dumps({os.environ.get('SKYRX_B200_SCORE_DEBUG', '0'): res}))
from paper_2602_13509_b200 import _lib, _dev
ds = plan.ds
def tc_only():
    _lib.call("skyrx_score_tc", raw.data_ptr(), L, S, B, d.data_ptr(), c.data_ptr(), None,
              ds.mu_hilo[0].data_ptr(), plan.wpack[0].data_ptr(), ds.flags[0:1].data_ptr(),
              plan.scores[0].data_ptr(), plan.max_key[0:1].data_ptr(), None, _dev.stream_ptr())
def topk_only():
    n = L * S
    _lib.call("skyrx_topk_threshold", plan.scores[0].data_ptr(), n, (n + 999) // 1000,
              plan.thr[0:1].data_ptr(), plan.topk_ws.data_ptr(), _dev.stream_ptr())
def mask_only():
    _lib.call("skyrx_mask_gt", plan.scores[0].data_ptr(), L * S, plan.thr[0:1].data_ptr(),
              plan.mask[0].data_ptr(), _dev.stream_ptr())
print(json.dumps({'tc_only_ms': t(tc_only), 'topk_ms': t(topk_only), 'mask_ms': t(mask_only)}))

def prep_only():
    _lib.call("skyrx_score_prep", ds.w64[0].data_ptr(), ds.mu_hilo[0].data_ptr(), S, B, d.data_ptr(),
              c.data_ptr(), 1.0, 1, plan.records[0].data_ptr(), _dev.stream_ptr())
def tcs_only():
    _lib.call("skyrx_score_tcs", raw.data_ptr(), L, S, B, plan.records[0].data_ptr(),
              ds.flags[0:1].data_ptr(), plan.scores[0].data_ptr(), plan.max_key[0:1].data_ptr(),
              None, _dev.stream_ptr())
if plan.tcs:
    print(json.dumps({'prep_ms': t(prep_only), 'tcs_only_ms': t(tcs_only)}))
print(json.dumps({'finalize_ms': t(lambda: plan.ds.finalize())}))
def shift_only():
    _lib.call("skyrx_stats_shift", _lib.IN_RAW_U16, raw.data_ptr(), L, S, B, d.data_ptr(), c.data_ptr(),
              g.data_ptr(), ds.shift[0].data_ptr(), _dev.stream_ptr())
print(json.dumps({'shift_ms': t(shift_only)}))
