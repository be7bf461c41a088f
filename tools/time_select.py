"""Select stage of one c4 strip: candidate count of skyrx_topk_mask and, under
`ncu --metrics gpu__time_duration.sum`, the per-kernel durations."""
import json, sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2602_13509_b200 as P
from paper_2602_13509_b200 import rx
from paper_2602_13509_b200.synth import Scene

L, S, B = 16384, 900, 70
sc = Scene(4000, S, B, 5)
raw = sc.generate(0, L)
d, c = torch.from_numpy(sc.dark).cuda(), torch.from_numpy(sc.coeff).cuda()
g = torch.ones(L, dtype=torch.float32, device='cuda')
plan = P.DetectPlan(L, S, B)
plan.run(0, raw, d, c, g, gain_const=1.0).finalize().score(0, raw, d, c, g)
torch.cuda.synchronize()
ncand = int(plan.topk_ws[1].item())
v = plan.scores[0].reshape(-1)
k = rx.topk_count(v.numel())
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
print(json.dumps({"ncand": ncand, "cap": plan.cand_cap, "k": k,
                  "one_pass_ms": t(lambda: rx.topk_mask_device(v, k)),
                  "threshold_ms": t(lambda: rx.topk_threshold_device(v, k))}))
