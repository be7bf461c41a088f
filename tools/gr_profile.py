"""Per-role wait breakdown of gram_raw_kernel.

Build a variant with the probes compiled in and run this against it:
    nvcc ... -DSKYRX_GR_PROFILE -c csrc/gram_raw.cu, relink, run.
"""
import ctypes, os, sys, json
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2602_13509_b200 as P
from paper_2602_13509_b200 import _lib
if os.environ.get('SKYRX_LIB'):
    _lib.load(os.environ['SKYRX_LIB'])
from paper_2602_13509_b200.synth import Scene
L, S, B = int(os.environ.get('GR_L', 16384)), 900, 70
sc = Scene(4000, S, B, 5)
raw = sc.generate(0, L)
d, c = torch.from_numpy(sc.dark).cuda(), torch.from_numpy(sc.coeff).cuda()
g = torch.ones(L, dtype=torch.float32, device='cuda')
plan = P.DetectPlan(L, S, B)
lib = _lib.load()
buf = (ctypes.c_ulonglong * (160 * 12))()
plan.run(0, raw, d, c, g, gain_const=1.0); torch.cuda.synchronize()
lib.skyrx_gr_profile(buf)
a0 = np.frombuffer(buf, dtype=np.uint64).reshape(160, 12).astype(np.float64).copy()
for _ in range(3):
    plan.run(0, raw, d, c, g, gain_const=1.0)
torch.cuda.synchronize()
lib.skyrx_gr_profile(buf)
a = (np.frombuffer(buf, dtype=np.uint64).reshape(160, 12).astype(np.float64) - a0)[:148] / 3
tot = a[:, 7].mean()
names = ['tma_wait_empty', 'mma_wait_acc_empty', 'mma_wait_full', 'scan_wait_full',
         'epi_wait_scan_full', 'epi_wait_acc_full', 'epi_active', 'total', 'epi_bands', 'epi_part0', 'epi_part01']
print(json.dumps({n: round(float(a[:, i].mean() / tot), 3) for i, n in enumerate(names)} | {'total_cycles': tot}))
