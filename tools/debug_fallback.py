"""Debug helper: the quantiser-range fallback path step by step."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2602_13509_b200 as P
from paper_2602_13509_b200 import _lib
from oracle import skyrx_oracle as O

rng = np.random.default_rng(20240901)
L, S, B = 60, 64, 70
raw = (1000 + rng.integers(-3, 4, (L, S, B))).astype(np.uint16)
raw[3, 5] = 4000
dark = np.full((S, B), 100.0, np.float32)
coeff = np.ones((S, B), np.float32)
rad = O.apply_calibration(raw, dark, coeff, np.ones(L))
ref = O.compute_stats(rad)
want = O.rx_scores(rad, ref)
rv = torch.from_numpy(raw).cuda()
d, c = torch.from_numpy(dark).cuda(), torch.from_numpy(coeff).cuda()
g = torch.ones(L, dtype=torch.float32, device='cuda')
for label, tc, ffma in [('tc stats', True, False), ('ffma stats', True, True), ('ffma+ffma', False, True)]:
    plan = P.DetectPlan(L, S, B)
    plan.tc = tc
    plan.run(0, rv, d, c, g, force_ffma=ffma).finalize().score(0, rv, d, c, g)
    torch.cuda.synchronize()
    st = int(plan.ds.status[0]); fl = int(plan.ds.flags[0])
    mu = plan.ds.mu[0].cpu().numpy(); sig = plan.ds.sigma[0].cpu().numpy()
    sc = plan.scores[0].cpu().numpy()
    rel = np.abs(sc - want) / want
    print(f'{label}: status {st} flags {fl} mu err {np.abs(mu-ref.mu).max():.3e} sigma err {np.abs(sig-ref.sigma).max()/np.abs(ref.sigma).max():.3e} '
          f'score max rel {rel.max():.3e} median {np.median(rel):.3e}')
