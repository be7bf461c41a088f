"""Is the cold-strip penalty of score_tc (0.49 -> 0.54 ms per c4 strip) the address
translation?  Cycle through N strips with / without touching one word per 64 KB / 2 MB of the
next strip just before its score launch, and cycle over 2 strips (4 GB)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2602_13509_b200 import _lib, _dev
import paper_2602_13509_b200 as P
from paper_2602_13509_b200.synth import Scene
L, S, B = 16384, 900, 70
N = 16
sc = Scene(4000, S, B, 5)
raws = [sc.generate(0, L) for _ in range(N)]
d, c = torch.from_numpy(sc.dark).cuda(), torch.from_numpy(sc.coeff).cuda()
g = torch.ones(L, dtype=torch.float32, device='cuda')
plan = P.DetectPlan(L, S, B)
plan.run(0, raws[0], d, c, g, gain_const=1.0).finalize().score(0, raws[0], d, c, g)
ds = plan.ds
sink = torch.zeros(1, dtype=torch.int64, device="cuda")
def tc(raw):
    _lib.call("skyrx_score_tc", raw.data_ptr(), L, S, B, d.data_ptr(), c.data_ptr(), None,
              ds.mu_hilo[0].data_ptr(), plan.wpack[0].data_ptr(), ds.flags[0:1].data_ptr(),
              plan.scores[0].data_ptr(), plan.max_key[0:1].data_ptr(), None, _dev.stream_ptr())
def touch(raw, stride_bytes):
    v = raw.view(-1).view(torch.int16)
    sink.add_(v[:: stride_bytes // 2].to(torch.int64).sum())
out = {}
for name, cyc, tstride in (("same", 1, 0), ("cycle2", 2, 0), ("cycle16", 16, 0),
                           ("cycle16_touch2M", 16, 2 << 20), ("cycle16_touch64K", 16, 64 << 10)):
    for _ in range(2):
        tc(raws[0])
    torch.cuda.synchronize()
    ms = 0.0
    for i in range(32):
        raw = raws[i % cyc]
        if tstride:
            touch(raw, tstride)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); tc(raw); b.record()
        torch.cuda.synchronize()
        ms += a.elapsed_time(b)
    out[name] = round(ms / 32, 4)
def gr(raw):
    plan.run(0, raw, d, c, g, gain_const=1.0)
for name, cyc in (("moments_same", 1), ("moments_cycle2", 2), ("moments_cycle16", 16)):
    for _ in range(2):
        gr(raws[0])
    torch.cuda.synchronize()
    ms = 0.0
    for i in range(32):
        raw = raws[i % cyc]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); gr(raw); b.record()
        torch.cuda.synchronize()
        ms += a.elapsed_time(b)
    out[name] = round(ms / 32, 4)
print(json.dumps(out))
