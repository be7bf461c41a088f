"""Latency of skyrx_stats_finalize (K3): panel (B <= 128), slot (B <= 80), wide (128 < B <= 288)
and general kernels.

    python tools/time_finalize.py   -> one line per (B, batch, kernel): us per call
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2602_13509_b200 as P  # noqa: E402

rng = np.random.default_rng(0)
for B in [int(b) for b in os.environ.get("BANDS", "16,70,128,270").split(",")]:
    for batch in (1, 64):
        n = 100000
        X = rng.standard_normal((4096, B)) @ np.diag(np.linspace(1, 30, B))
        q = X.T @ X * (n / 4096)
        mom = np.concatenate([[float(n)], X.sum(0) * 0, q.ravel()])
        ds = P.DeviceStats(B, batch=batch)
        ds.moments.copy_(torch.from_numpy(np.tile(mom, (batch, 1))))
        for kind in ("panel", "slot", "general"):
            os.environ.pop("SKYRX_B200_FIN_GENERAL", None)
            os.environ.pop("SKYRX_B200_FIN_SLOT", None)
            if kind == "general":
                os.environ["SKYRX_B200_FIN_GENERAL"] = "1"
            elif kind == "slot":
                if B > 80:
                    continue
                os.environ["SKYRX_B200_FIN_SLOT"] = "1"
            for _ in range(3):
                ds.finalize()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                ds.finalize()
            b.record()
            torch.cuda.synchronize()
            print(f"B={B} batch={batch} {kind:8s}: "
                  f"{a.elapsed_time(b) / 20 * 1e3:.1f} us per call", flush=True)
