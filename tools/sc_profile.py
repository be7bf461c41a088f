"""Per-role wait breakdown of score_tc_kernel (build: tools/build_sc_var.sh prof
-DSKYRX_SC_PROFILE; run: python tools/sc_profile.py tools/_var/prof.so)."""
import ctypes, json, sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2602_13509_b200 import _lib, _dev
_lib.load(sys.argv[1])
import paper_2602_13509_b200 as P
from paper_2602_13509_b200.synth import Scene
L, S, B = 16384, 900, 70
sc = Scene(4000, S, B, 5)
raw = sc.generate(0, L)
d, c = torch.from_numpy(sc.dark).cuda(), torch.from_numpy(sc.coeff).cuda()
g = torch.ones(L, dtype=torch.float32, device='cuda')
plan = P.DetectPlan(L, S, B)
plan.run(0, raw, d, c, g, gain_const=1.0).finalize()
ds = plan.ds
lib = _lib.load()
def fn():
    _lib.call("skyrx_score_tc", raw.data_ptr(), L, S, B, d.data_ptr(), c.data_ptr(), None,
              ds.mu_hilo[0].data_ptr(), plan.wpack[0].data_ptr(), ds.flags[0:1].data_ptr(),
              plan.scores[0].data_ptr(), plan.max_key[0:1].data_ptr(), None, _dev.stream_ptr())
buf = (ctypes.c_ulonglong * (160 * 10))()
fn(); torch.cuda.synchronize()
lib.skyrx_sc_profile(buf)
a0 = np.frombuffer(buf, dtype=np.uint64).reshape(160, 10).astype(np.float64).copy()
for _ in range(3): fn()
torch.cuda.synchronize()
lib.skyrx_sc_profile(buf)
a = (np.frombuffer(buf, dtype=np.uint64).reshape(160, 10).astype(np.float64) - a0)[:148] / 3
tot = a[:, 9].mean()
per = {'xf_wait_raw_full': (0, 12), 'xf_wait_a_empty': (1, 12), 'xf_compute': (2, 12),
       'xf_tmem_st_wait': (3, 12), 'mma_wait_a_full': (4, 1), 'mma_wait_acc_empty': (5, 1),
       'epi_wait_acc_full': (6, 4)}
print(json.dumps({k: round(float(a[:, i].mean() / n / tot), 3) for k, (i, n) in per.items()}
                 | {'total_cycles': tot}))
