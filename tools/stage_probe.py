"""Per-stage device+host time of the air pipeline's work on one paper-geometry cube
(1000 x 900 x 300 raw -> 70 bands), run back to back on one stream."""
import time

import numpy as np
import torch

import paper_2602_13509_b200 as P
from paper_2602_13509_b200 import datalink as D, synth

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
host = torch.empty(raw.shape, dtype=torch.uint16, pin_memory=True)
host.copy_(raw)


def t(label, fn, n=10):
    out = fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        out = fn()
    torch.cuda.synchronize()
    print(f"{label}: {(time.perf_counter() - t0) / n * 1e3:.2f} ms")
    return out


t("H2D pinned raw", lambda: host.to("cuda", non_blocking=True))
binned, rgb = t("calibrate_bin_rgb", lambda: P.calibrate_bin_rgb(cube, tables, factor=4))
for mode in ("precise", "fast"):
    st = t(f"compute_stats {mode}", lambda: P.compute_stats(binned, mode=mode))
    sc = t(f"rx_scores {mode}", lambda: P.rx_scores(binned, st, mode=mode))
t("cube_frames", lambda: D.cube_frames(1, rgb, sc.values, metas))
