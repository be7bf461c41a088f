"""H2D / D2H bandwidth probe: pinned torch tensor, numpy view of pinned, pageable numpy."""
import time, json, numpy as np, torch
n = 1 << 30
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
pin = torch.empty(n, dtype=torch.uint8, pin_memory=True)
pin.fill_(1)
page = np.ones(n, np.uint8)
res = {}
def t(name, fn, reps=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    res[name] = round(n * reps / (time.perf_counter() - t0) / 1e9, 1)
t("h2d_pinned_tensor", lambda: dev.copy_(pin, non_blocking=True))
t("h2d_numpy_view_of_pinned", lambda: dev.copy_(torch.from_numpy(pin.numpy()), non_blocking=True))
t("h2d_numpy_to", lambda: torch.from_numpy(pin.numpy()).to("cuda"))
t("h2d_pageable", lambda: dev.copy_(torch.from_numpy(page)))
t("d2h_pinned", lambda: pin.copy_(dev, non_blocking=True))
t("d2h_pageable", lambda: dev.cpu())
res["from_numpy_is_pinned"] = torch.from_numpy(pin.numpy()).is_pinned()
print(json.dumps(res))
