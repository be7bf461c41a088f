"""One batched finalize (148 matrices, B from argv) for an ncu source-level capture."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2602_13509_b200 as P  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 70
rng = np.random.default_rng(0)
n = 100000
X = rng.standard_normal((4096, B)) @ np.diag(np.linspace(1, 30, B))
mom = np.concatenate([[float(n)], X.sum(0) * 0, (X.T @ X * (n / 4096)).ravel()])
ds = P.DeviceStats(B, batch=148)
ds.moments.copy_(torch.from_numpy(np.tile(mom, (148, 1))))
for _ in range(3):
    ds.finalize()
torch.cuda.synchronize()
print("ok", int(ds.status.sum().item()))
