"""Debug helper: compare tensor-core moments with the oracle on one small cube."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2602_13509_b200 as P
from paper_2602_13509_b200 import _lib, _dev
from oracle import synth as osynth, skyrx_oracle as O

S, B, L = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
t = osynth.make_tables(43, S, B, 5)
raw = osynth.generate_lines(t, 0, L)
rv = torch.from_numpy(raw).cuda()
dark, coeff = torch.from_numpy(t.dark).cuda(), torch.from_numpy(t.coeff).cuda()
g = torch.ones(L, dtype=torch.float32, device='cuda')
plan = P.DetectPlan(L, S, B)
plan.run(0, rv, dark, coeff, g)
torch.cuda.synchronize()
m = plan.ds.moments[0].cpu().numpy()
shift = plan.ds.shift[0].cpu().numpy()
qinv = plan.qinv[0].cpu().numpy()
print('flags', plan.ds.flags.cpu().numpy(), 'qinv range', qinv.min(), qinv.max())
rad = O.apply_calibration(raw, t.dark, t.coeff, np.ones(L)).reshape(-1, B)
n, s, Q = O.moments(rad, shift)
print('n', m[0], n)
print('s err', np.abs(m[1:1+B] - s).max(), 'scale', np.abs(s).max())
Qd = m[1+B:].reshape(B, B)
err = np.abs(Qd - Q)
print('Q err max', err.max(), 'scale', np.abs(Q).max())
i, j = np.unravel_index(err.argmax(), err.shape)
print('worst at', i, j, Qd[i, j], Q[i, j])
print('diag ratio', (np.diag(Qd) / np.diag(Q))[:10])
print('row0', Qd[0, :6], Q[0, :6])
