"""Where does the host-buffer detect() time go?  (one c4 strip, pinned host input)"""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2602_13509_b200 as P
from paper_2602_13509_b200 import _dev, rx
from paper_2602_13509_b200.synth import Scene
L, S, B = 16384, 900, 70
sc = Scene(4000, S, B, 5)
host = sc.generate(0, L).cpu().pin_memory().numpy()
cube = P.RawCube(host, np.linspace(400, 1000, B), gains=np.ones(L, np.float32))
tab = P.CalibrationTables(sc.dark, sc.coeff)
plan = P.DetectPlan(L, S, B)
for _ in range(2):
    det = P.detect(cube, tab, plan=plan)
torch.cuda.synchronize()
T = {}
def tic(): torch.cuda.synchronize(); return time.perf_counter()
t0 = tic(); rv = rx._raw_device(cube); t1 = tic(); T['h2d_raw'] = t1 - t0
t0 = tic(); det = P.detect(cube, tab, plan=plan); t1 = tic(); T['detect_total'] = t1 - t0
t0 = tic(); s = _dev.to_host(plan.scores[0]); t1 = tic(); T['d2h_scores'] = t1 - t0
t0 = tic(); m = _dev.to_host(plan.mask[0]); t1 = tic(); T['d2h_mask'] = t1 - t0
t0 = tic(); st = plan.ds.host(0, L * S); t1 = tic(); T['stats_host'] = t1 - t0
print(json.dumps({k: round(v * 1e3, 2) for k, v in T.items()}))
