"""The air pipeline's device work on one paper-geometry cube (1000 x 900 x 300 raw ->
70 bands): calibrate_bin_rgb, compute_stats / rx_scores in both modes, frames.
For `ncu --metrics gpu__time_duration.sum` launch lists (tools/r2_air_kernels.sh)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2602_13509_b200 as P  # noqa: E402
from paper_2602_13509_b200 import synth  # noqa: E402

L, S, B = 1000, 900, 300
inner = np.linspace(400.0, 1000.0, B - 20)
step = inner[1] - inner[0]
wl = np.concatenate([400.0 - step * np.arange(10, 0, -1), inner, 1000.0 + step * np.arange(1, 11)])
scene = synth.Scene(7, S, B)
raw = scene.generate(0, L)
ins = P.InsSample(5, 35.0, -90.0, 40.0, 0.0, 0.0, 0.0)
metas = [P.LineMeta(i, 1.0 + 0.125 * (i % 4), ins, ins) for i in range(L)]
cube = P.RawCube(raw, wl, metas)
tables = P.CalibrationTables(scene.dark, scene.coeff)
for _ in range(2):
    binned, rgb = P.calibrate_bin_rgb(cube, tables, factor=4)
    for mode in ("precise", "fast"):
        st = P.compute_stats(binned, mode=mode)
        sc = P.rx_scores(binned, st, mode=mode)
torch.cuda.synchronize()
print("ok", binned.values.shape)
