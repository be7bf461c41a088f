"""One DetectPlan step (moments + finalize + scores + mask) on a seeded cube, CUDA events,
optionally through another build of the library (variant experiments).
    python tools/time_plan.py L S B [lib.so]"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2602_13509_b200 import _lib  # noqa: E402

L, S, B = (int(x) for x in sys.argv[1:4])
if len(sys.argv) > 4:
    _lib.load(sys.argv[4])
import paper_2602_13509_b200 as P  # noqa: E402
from paper_2602_13509_b200.synth import Scene  # noqa: E402

sc = Scene(4000, S, B, 8)
raw = sc.generate(0, L)
d, c = torch.from_numpy(sc.dark).cuda(), torch.from_numpy(sc.coeff).cuda()
g = torch.ones(L, dtype=torch.float32, device="cuda")
plan = P.DetectPlan(L, S, B)
for _ in range(3):
    plan.run(0, raw, d, c, g, gain_const=1.0)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    plan.run(0, raw, d, c, g, gain_const=1.0)
b.record()
torch.cuda.synchronize()
print(f"{sys.argv[4] if len(sys.argv) > 4 else 'product'}: {a.elapsed_time(b) / 5:.3f} ms per step, "
      f"flags {int(plan.ds.flags[0].item())}")
