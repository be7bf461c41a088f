"""calibrate_bin_rgb at paper geometry (1000 x 900 x 300 raw -> 70 bands + RGB), CUDA events.
    python tools/time_calbin.py [lib.so]  -> us per cube and GB/s of N (2B + 4B') + RGB"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2602_13509_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.load(sys.argv[1])
import paper_2602_13509_b200 as P  # noqa: E402
from paper_2602_13509_b200 import synth  # noqa: E402

L, S, B = 1000, 900, 300
inner = np.linspace(400.0, 1000.0, B - 20)
step = inner[1] - inner[0]
wl = np.concatenate([400.0 - step * np.arange(10, 0, -1), inner, 1000.0 + step * np.arange(1, 11)])
scene = synth.Scene(7, S, B)
raw = scene.generate(0, L)  # device tensor
ins = P.InsSample(5, 35.0, -90.0, 40.0, 0.0, 0.0, 0.0)
metas = [P.LineMeta(i, 1.0 + 0.125 * (i % 4), ins, ins) for i in range(L)]
cube = P.RawCube(raw, wl, metas)
tables = P.CalibrationTables(scene.dark, scene.coeff)
for _ in range(3):
    binned, rgb = P.calibrate_bin_rgb(cube, tables, factor=4)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 20
a.record()
for _ in range(n):
    binned, rgb = P.calibrate_bin_rgb(cube, tables, factor=4)
b.record()
torch.cuda.synchronize()
us = a.elapsed_time(b) / n * 1e3
nb = binned.values.shape[-1]
byt = L * S * (2 * B + 4 * nb + 12)
print(f"calibrate_bin_rgb {L}x{S}x{B} -> {nb}: {us:.1f} us per cube (incl. host-side call), "
      f"{byt / us / 1e3:.0f} GB/s")
