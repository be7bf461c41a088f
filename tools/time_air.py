"""Air pipeline at paper geometry: N cubes of 1000 x 900 x 300 raw (host, pinned or
.hsc files) through air.run_air (calibrate+bin -> moments/factor/scores -> packets+RS parity
-> frames).  Prints cubes/s, per-stage times, and the same for .hsc ingest."""
import sys
import tempfile
import time
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import torch

import paper_2602_13509_b200 as P
from paper_2602_13509_b200 import formats, synth
from paper_2602_13509_b200.air import run_air

n_cubes = int(sys.argv[1]) if len(sys.argv) > 1 else 8
L, S, B = 1000, 900, 300
inner = np.linspace(400.0, 1000.0, B - 20)
step = inner[1] - inner[0]
wl = np.concatenate([400.0 - step * np.arange(10, 0, -1), inner, 1000.0 + step * np.arange(1, 11)])
wl = wl.astype(np.float32).astype(np.float64)
scene = synth.Scene(7, S, B)
ins = P.InsSample(5, 35.0, -90.0, 40.0, 0.0, 0.0, 0.0)
cubes = []
for c in range(n_cubes):
    raw = scene.generate(c * L, L)
    host = torch.empty(raw.shape, dtype=torch.uint16, pin_memory=True)
    host.copy_(raw)
    metas = [P.LineMeta(c * 10**6 + i, 1.0 + 0.125 * (i % 4), ins, ins) for i in range(L)]
    cubes.append(P.RawCube(host, wl, metas))
torch.cuda.synchronize()
tables = P.CalibrationTables(scene.dark, scene.coeff)
cfg = SimpleNamespace(bin_factor=4, queue_depth=3, out_dir=None)


def go(data, label):
    run_air(cfg, SimpleNamespace(cubes=data[:2], tables=tables))   # warm-up
    t0 = time.perf_counter()
    res = run_air(cfg, SimpleNamespace(cubes=data, tables=tables))
    dt = time.perf_counter() - t0
    st = np.array([t.as_tuple() for t in res.timings]).mean(axis=0) * 1e3
    print(f"{label}: {len(data)} cubes in {dt:.3f} s = {len(data) / dt:.2f} cubes/s "
          f"({len(data) * L * S / dt / 1e6:.1f} Mpx/s); stage ms save/cal/det/tx = "
          f"{st[0]:.1f}/{st[1]:.1f}/{st[2]:.1f}/{st[3]:.1f}; frames {len(res.frames)}; "
          f"dropped {res.dropped}")
    return res


r1 = go(cubes, "pinned host cubes")
with tempfile.TemporaryDirectory() as td:
    paths = []
    for i, c in enumerate(cubes):
        p = Path(td) / f"cube_{i:04d}.hsc"
        formats.write_cube(p, c)
        paths.append(p)
    r2 = go(paths, ".hsc ingest")
print("same stream:", r1.frames == r2.frames)
