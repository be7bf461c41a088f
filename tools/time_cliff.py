"""Fast path vs the clamp-corrected path on full c4 strips (verdict #7: the fallback
should cost <= 1.3x the fast path).  0.01 % random sub-dark counts, and one dead
detector element, and sinusoidal per-line gains (the quantised-digit
tensor-core moments); CUDA events around moments + finalize + scores + mask per strip.

    python tools/time_cliff.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2602_13509_b200 import _dev  # noqa: E402
from paper_2602_13509_b200.strips import StripBatch  # noqa: E402
from paper_2602_13509_b200.synth import Scene  # noqa: E402

L, S, B = 16384, 900, 70
sc = Scene(4000, S, B, 5)
clean = sc.generate(0, L)
g = torch.Generator(device="cuda").manual_seed(1)
sparse = clean.clone()
flat = sparse.view(torch.int16).view(-1)
idx = torch.randint(0, flat.numel(), (flat.numel() // 10000,), device="cuda", generator=g)
flat[idx] = 7
dead = clean.clone()
dead.view(torch.int16)[:, 300, 35] = 5
tabs = [(_dev.to_device(sc.dark), _dev.to_device(sc.coeff))]
ones = [_dev.to_device(np.ones(L, np.float32))]
# per-line gains varying like the reference scene's exposure drift (a slow sinusoid)
sinus = [_dev.to_device((1.0 + 0.05 * np.sin(np.arange(L) * 2 * np.pi / 977.0)).astype(np.float32))]
cases = (("clean", clean, ones, 1.0), ("0.01% sub-dark", sparse, ones, 1.0),
         ("dead element", dead, ones, 1.0), ("sinusoidal gains", clean, sinus, None))
for name, raw, gains, gconst in cases:
    b = StripBatch(L, S, B, 1)
    for _ in range(3):
        b.enqueue([raw], tabs, gains, [gconst])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        b.enqueue([raw], tabs, gains, [gconst])
    e1.record()
    torch.cuda.synchronize()
    st, fl = b.flags()
    print(f"{name:16s}: {e0.elapsed_time(e1) / 10:.3f} ms per strip, status {st[0]}, "
          f"flags {int(fl[0])}", flush=True)
