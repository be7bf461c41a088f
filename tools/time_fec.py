"""Time the downlink kernels on one 1000 x 900 cube: link maxima + packets, RS parity of its
20 groups (50 x 3728 B each), and batched erasure recovery of 20 groups with 25 erasures."""
import time

import numpy as np
import torch

import paper_2602_13509_b200 as P
from paper_2602_13509_b200 import datalink as D, fec as F
from oracle import skyrx_oracle as O


def timeit(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


rng = np.random.default_rng(0)
lines = 1000
rgb = torch.from_numpy((rng.random((lines, 900, 3)) * 30).astype(np.float32)).cuda()
sc = torch.from_numpy((rng.random((lines, 900)) ** 4 * 900).astype(np.float32)).cuda()
ins = P.InsSample(5, 35.0, -90.0, 40.0, 0.0, 0.0, 0.0)
metas = [P.LineMeta(1000 + i, 1.0, ins, ins) for i in range(lines)]
pk = D.cube_packets(1, rgb, sc, metas)
code = D._codec()
data = pk.view(20, 50, -1)
par = code.encode_groups(data)
us_pk = timeit(lambda: D.cube_packets(1, rgb, sc, metas), 10)
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    code.encode_groups(data, out=par)
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            code.encode_groups(data, out=par)
torch.cuda.current_stream().wait_stream(s)
us_par = timeit(g.replay, 10) / 20  # graph replays: device time, no host launch overhead
nbytes = data.numel() + par.numel()
print(f"cube_packets (incl. host headers): {us_pk:.1f} us")
print(f"RS parity 20 groups: {us_par:.1f} us  ({nbytes / us_par / 1e3:.1f} GB/s of data+parity)")
# recovery: 20 groups, each missing 25 random data slots (worst case for the matmul)
host = pk.cpu().numpy().reshape(20, 50, -1)
parh = par.cpu().numpy()
groups = []
for g in range(20):
    coded = [host[g, i].tobytes() for i in range(50)] + [parh[g, i].tobytes() for i in range(25)]
    keep = sorted(rng.permutation(75)[:50])
    groups.append([(int(i), coded[i]) for i in keep])
t0 = time.perf_counter()
res = code.decode_groups(groups)
torch.cuda.synchronize()
t1 = time.perf_counter()
ok = all(b"".join(r[0][i] for i in range(50)) == host[g].tobytes() for g, r in enumerate(res))
print(f"decode_groups 20 groups (host wall incl. H2D/D2H): {(t1 - t0) * 1e3:.2f} ms ok={ok}")
t0 = time.perf_counter()
O.rs_encode(O.encoding_matrix(50, 75), 50, [host[0, i].tobytes() for i in range(50)])
t1 = time.perf_counter()
print(f"oracle numpy parity of ONE group: {(t1 - t0) * 1e3:.1f} ms")
