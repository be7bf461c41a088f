"""Debug helper: isolate TC score error with precise (f64) statistics."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2602_13509_b200 as P
from oracle import synth as osynth, skyrx_oracle as O

S, B, L = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
t = osynth.make_tables(41, S, B, 5)
raw = osynth.generate_lines(t, 0, L)
rv = torch.from_numpy(raw).cuda()
dark, coeff = torch.from_numpy(t.dark).cuda(), torch.from_numpy(t.coeff).cuda()
g = torch.ones(L, dtype=torch.float32, device='cuda')
rad = O.apply_calibration(raw, t.dark, t.coeff, np.ones(L))
ref = O.compute_stats(rad)
want = O.rx_scores(rad, ref)
for tc in (True, False):
    for precise in (True, False):
        plan = P.DetectPlan(L, S, B)
        plan.tc = tc
        plan.run(0, rv, dark, coeff, g, precise=precise).finalize().score(0, rv, dark, coeff, g)
        torch.cuda.synchronize()
        sc = plan.scores[0].cpu().numpy()
        rel = np.abs(sc - want) / want
        i = np.unravel_index(rel.argmax(), rel.shape)
        sig = plan.ds.sigma[0].cpu().numpy()
        print(f'tc={tc} precise={precise}: max rel {rel.max():.3e} at {i} got {sc[i]:.6g} want {want[i]:.6g}; '
              f'median {np.median(rel):.2e}; sigma err {np.abs(sig-ref.sigma).max()/np.abs(ref.sigma).max():.2e}')
        bad = rel > 1e-4
        if bad.any():
            ls, ss = np.nonzero(bad)
            print('   bad count', bad.sum(), 'lines', np.unique(ls)[:10], 'samples', np.unique(ss)[:20])
