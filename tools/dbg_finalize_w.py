import os, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2602_13509_b200 as P
B = int(sys.argv[1])
rng = np.random.default_rng(B)
X = rng.standard_normal((5000, B)) @ np.diag(np.linspace(1, 30, B)) + 50
c = X[:64].mean(0); d = X - c
mom = np.concatenate([[5000.0], d.sum(0), (d.T @ d).ravel()])
out = {}
for gen in (0, 1):
    if gen: os.environ["SKYRX_B200_FIN_GENERAL"] = "1"
    else: os.environ.pop("SKYRX_B200_FIN_GENERAL", None)
    ds = P.DeviceStats(B, batch=1)
    ds.moments.copy_(torch.from_numpy(mom[None])); ds.shift.copy_(torch.from_numpy(c[None]))
    ds.finalize(); torch.cuda.synchronize()
    out[gen] = (ds.w64[0].cpu().numpy(), ds.chol[0].cpu().numpy())
w0, w1 = out[0][0], out[1][0]
diff = np.argwhere(w0 != w1)
print(B, "ndiff", len(diff), diff[:10].tolist(), "chol equal", np.array_equal(out[0][1], out[1][1]))
if len(diff):
    i, j = diff[0]
    print(w0[i, j], w1[i, j], np.abs(w0 - w1).max() / np.abs(w1).max())
