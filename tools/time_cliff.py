"""Fast path vs the clamp-corrected path on full c4 strips (verdict #7: the fallback
should cost <= 1.3x the fast path).  0.01 % random sub-dark counts, and one dead
detector element; CUDA events around moments + finalize + scores + mask per strip.

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
gains = [_dev.to_device(np.ones(L, np.float32))]
for name, raw in (("clean", clean), ("0.01% sub-dark", sparse), ("dead element", dead)):
    b = StripBatch(L, S, B, 1)
    for _ in range(3):
        b.enqueue([raw], tabs, gains, [1.0])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        b.enqueue([raw], tabs, gains, [1.0])
    e1.record()
    torch.cuda.synchronize()
    st, fl = b.flags()
    print(f"{name:16s}: {e0.elapsed_time(e1) / 10:.3f} ms per strip, status {st[0]}, "
          f"flags {int(fl[0])}", flush=True)
