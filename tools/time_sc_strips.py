"""score_tc on the same c4 strip repeated vs cycling through N different strips (CUDA events):
does touching a fresh 2 GB strip (TLB / DRAM page state) cost per-launch time?"""
import json, os, sys
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2602_13509_b200 import _lib, _dev
import paper_2602_13509_b200 as P
from paper_2602_13509_b200.synth import Scene
L, S, B = 16384, 900, 70
N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
sc = Scene(4000, S, B, 5)
raws = [sc.generate(0, L) for _ in range(N)]
d, c = torch.from_numpy(sc.dark).cuda(), torch.from_numpy(sc.coeff).cuda()
g = torch.ones(L, dtype=torch.float32, device='cuda')
plan = P.DetectPlan(L, S, B)
plan.run(0, raws[0], d, c, g, gain_const=1.0).finalize().score(0, raws[0], d, c, g)
ds = plan.ds
def tc(raw):
    _lib.call("skyrx_score_tc", raw.data_ptr(), L, S, B, d.data_ptr(), c.data_ptr(), None,
              ds.mu_hilo[0].data_ptr(), plan.wpack[0].data_ptr(), ds.flags[0:1].data_ptr(),
              plan.scores[0].data_ptr(), plan.max_key[0:1].data_ptr(), None, _dev.stream_ptr())
def gr(raw):
    plan.run(0, raw, d, c, g, gain_const=1.0)
out = {}
for name, fn in (("score_tc", tc), ("moments", gr)):
    for mode in ("same", "cycle"):
        for _ in range(2):
            fn(raws[0])
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(4 * N):
            fn(raws[0] if mode == "same" else raws[i % N])
        b.record(); torch.cuda.synchronize()
        out[f"{name}_{mode}"] = round(a.elapsed_time(b) / (4 * N), 4)
print(json.dumps(out))
