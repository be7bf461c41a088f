"""Experiment: the moments pass of strip B beside the score pass of strip A on
disjoint halves of the SMs (two streams), against the two passes back to back
on all SMs.  Needs a library built with -DGRX_NSPLIT_ENV -DSCX_GRID_ENV."""
import json, os, sys
import torch
sys.path.insert(0, '.')
from paper_2602_13509_b200 import _lib, _dev
_lib.load(sys.argv[1])
import paper_2602_13509_b200 as P
from paper_2602_13509_b200.synth import Scene
L, S, B = 16384, 900, 70
scs = [Scene(4000 + i, S, B, 5) for i in range(2)]
raws = [sc.generate(0, L) for sc in scs]
tabs = [(torch.from_numpy(sc.dark).cuda(), torch.from_numpy(sc.coeff).cuda()) for sc in scs]
g = torch.ones(L, dtype=torch.float32, device='cuda')
plan = P.DetectPlan(L, S, B, batch=2)
for j in range(2):
    plan.run(j, raws[j], *tabs[j], g, gain_const=1.0)
plan.finalize()
torch.cuda.synchronize()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def pair(split):
    os.environ["SKYRX_GR_GRID"] = "74" if split else "148"
    os.environ["SKYRX_SC_GRID"] = "74" if split else "148"
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(); e2 = torch.cuda.Event()
    cur = torch.cuda.current_stream()
    a.record(cur)
    s1.wait_stream(cur); s2.wait_stream(cur)
    for rep in range(8):
        with torch.cuda.stream(s1):
            plan.run(1, raws[1], *tabs[1], g, gain_const=1.0)
        st = s2 if split else s1
        with torch.cuda.stream(st):
            plan.score_only(0, raws[0], *tabs[0], g)
    e1.record(s1); e2.record(s2)
    cur.wait_event(e1); cur.wait_event(e2)
    b.record(cur)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 8
pair(False); pair(True)
res = {"back_to_back_full_grid_ms": pair(False), "concurrent_halves_ms": pair(True),
       "back_to_back_again_ms": pair(False), "concurrent_again_ms": pair(True)}
print(json.dumps(res))
