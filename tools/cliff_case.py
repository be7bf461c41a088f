"""One c4 strip with 0.01 % sub-dark counts (or a dead element with --dead) through
StripBatch, for an ncu launch list of the clamp-corrected path."""
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
raw = sc.generate(0, L)
gconst = 1.0
gains = [_dev.to_device(np.ones(L, np.float32))]
if "--dead" in sys.argv:
    raw.view(torch.int16)[:, 300, 35] = 5
elif "--gains" in sys.argv:  # sinusoidal per-line gains: quantised-digit moments
    gains = [_dev.to_device((1.0 + 0.05 * np.sin(np.arange(L) * 2 * np.pi / 977.0)).astype(np.float32))]
    gconst = None
else:
    g = torch.Generator(device="cuda").manual_seed(1)
    flat = raw.view(torch.int16).view(-1)
    flat[torch.randint(0, flat.numel(), (flat.numel() // 10000,), device="cuda", generator=g)] = 7
tabs = [(_dev.to_device(sc.dark), _dev.to_device(sc.coeff))]
b = StripBatch(L, S, B, 1)
for _ in range(2):
    b.enqueue([raw], tabs, gains, [gconst])
torch.cuda.synchronize()
print("flags", b.flags())
