"""R-GLOBAL CUDA ops on the GPU.

(1) world_size 1: distributed.global_detect with the CUDA ops equals the
    single-cube detect path and the oracle.
(2) two line blocks on one GPU with the collectives done by hand (sums /
    max of the tensors the protocol would all-reduce; no kernel waits on
    another): equals the oracle on the concatenated cube — the CUDA-side
    composition the NCCL run relies on.
"""

import numpy as np
import pytest

from oracle import skyrx_oracle as O
from oracle import synth as osynth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2602_13509_b200 as P
    from paper_2602_13509_b200 import build

    build.build()
    return P


def normwise(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300)


@pytest.mark.parametrize("seed,L,S,B", [(5, 64, 96, 70), (5, 40, 64, 128), (8, 30, 40, 16)])
def test_single_rank_global_equals_detect(P, seed, L, S, B):
    from paper_2602_13509_b200.distributed import GlobalRX

    t = osynth.make_tables(seed, S, B, 5)
    raw = osynth.generate_lines(t, 0, L)
    tabs = P.CalibrationTables(t.dark, t.coeff)
    g = GlobalRX(L, S, B, tabs, n_total=L * S).detect(raw)
    want_stats, want_scores, want_mask = O.detect(raw, t.dark, t.coeff, np.ones(L))
    assert normwise(g.stats.mu, want_stats.mu) < 1e-5
    assert normwise(g.stats.sigma, want_stats.sigma) < 1e-5
    sc = g.scores.cpu().numpy()
    assert (np.abs(sc - want_scores) / np.maximum(want_scores, 1e-12)).max() < 1e-4
    thr = O.topk_threshold(want_scores)
    near = np.abs(want_scores - thr) <= 1e-4 * abs(thr)
    assert not ((g.mask.cpu().numpy() != want_mask) & ~near).any()
    # the split top-k steps reproduce the one-call select on the same scores
    assert g.threshold == O.topk_threshold(sc)
    assert g.max_score == float(sc.max())


@pytest.mark.parametrize("seed,L,S,B", [(5, 64, 96, 70), (5, 48, 64, 128)])
def test_two_blocks_by_hand_equal_oracle(P, seed, L, S, B):
    import torch
    from paper_2602_13509_b200 import _dev
    from paper_2602_13509_b200.distributed import CudaOps

    t = osynth.make_tables(seed, S, B, 5)
    tabs = P.CalibrationTables(t.dark, t.coeff)
    half = L // 2
    raws = [_dev.to_device(osynth.generate_lines(t, r * half, half), torch.uint16)
            for r in range(2)]
    ops = [CudaOps(half, S, B, tabs) for _ in range(2)]
    n_total = L * S
    shift = ops[0].shift(raws[0]).clone()
    parts = [op.moments(raw, shift) for op, raw in zip(ops, raws)]
    mom = parts[0][0].clone() + parts[1][0]
    nonfin = torch.maximum(parts[0][1], parts[1][1])
    for op, (m, _) in zip(ops, parts):
        m.copy_(mom)
    stats = [op.check(op.finalize(mom, shift, nonfin), n_total) for op in ops]
    assert np.array_equal(stats[0].sigma_inv, stats[1].sigma_inv)
    scores = [op.score(raw)[0] for op, raw in zip(ops, raws)]
    k = O.topk_count(n_total)
    for op in ops:
        op.topk_init(n_total, k)
    for digit in range(3):
        hs = [op.topk_hist(sc, digit) for op, sc in zip(ops, scores)]
        tot = hs[0].clone() + hs[1]
        for h in hs:
            h.copy_(tot)
        for op in ops:
            op.topk_pick(digit)
    thr = [op.threshold() for op in ops]
    assert thr[0] == thr[1]
    allsc = np.concatenate([s.cpu().numpy() for s in scores])
    assert thr[0] == O.topk_threshold(allsc)
    masks = np.concatenate([op.mask(sc).cpu().numpy() for op, sc in zip(ops, scores)])
    assert np.array_equal(masks, O.topk_mask(allsc))
    raw = osynth.generate_lines(t, 0, L)
    want = O.compute_stats(O.apply_calibration(raw, t.dark, t.coeff, np.ones(L)))
    assert normwise(stats[0].mu, want.mu) < 1e-5
    assert normwise(stats[0].sigma, want.sigma) < 1e-5
    wsc = O.rx_scores(O.apply_calibration(raw, t.dark, t.coeff, np.ones(L)), want)
    assert (np.abs(allsc - wsc) / np.maximum(wsc, 1e-12)).max() < 1e-4
