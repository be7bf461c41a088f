"""The multi-strip path (BASELINE config 4) on the GPU: StripBatch / detect_strips.

One batched plan per rank (moments of every strip, one batched finalize,
scores + masks) must return, strip by strip, exactly what detect() returns
for that strip alone — including a strip that clamps (redone through the
general kernels by verify()) — and a CUDA-graph replay of enqueue() must
equal the eager launch bit for bit (bench.py times the replay).
"""

import numpy as np
import pytest

from oracle import synth as osynth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2602_13509_b200 as P
    from paper_2602_13509_b200 import build

    build.build()
    return P


def strips(P, n, L=600, S=900, B=70, clamp=None):
    out = []
    for i in range(n):
        t = osynth.make_tables(500 + i, S, B, 5)
        raw = osynth.generate_lines(t, 0, L).copy()
        if i == clamp:
            raw[7, 11, 3] = 0       # below dark: the fast moments cannot take it
        out.append((P.RawCube(raw, np.linspace(400, 1000, B), gains=np.ones(L, np.float32)),
                    P.CalibrationTables(t.dark, t.coeff)))
    return out


def test_detect_strips_equals_detect_per_strip(P):
    src = strips(P, 4, clamp=2)
    res = P.detect_strips(src)
    assert res.world == 1 and sorted(res.local) == [0, 1, 2, 3]
    assert [s.index for s in res.summary] == [0, 1, 2, 3]
    for i, (raw, tab) in enumerate(src):
        got, want = res.local[i], P.detect(raw, tab)
        assert np.array_equal(got.scores.view(np.uint32), want.scores.view(np.uint32)), i
        assert np.array_equal(got.mask, want.mask), i
        assert got.threshold == want.threshold and got.max_score == want.max_score
        assert np.array_equal(got.stats.sigma_inv, want.stats.sigma_inv), i
        assert res.summary[i].anomalies == int(want.mask.sum())


def test_callable_source_and_device_results(P):
    import torch

    src = strips(P, 3)
    res = P.detect_strips(lambda i: src[i], 3, host=False)
    assert isinstance(res.local[1].scores, torch.Tensor) and res.local[1].scores.is_cuda
    want = P.detect(*src[1])
    assert np.array_equal(res.local[1].scores.cpu().numpy(), want.scores)


def test_graph_replay_equals_eager_and_flags_checked(P):
    import torch
    from paper_2602_13509_b200 import _dev
    from paper_2602_13509_b200.strips import StripBatch, needs_redo
    from paper_2602_13509_b200.synth import Scene

    L, S, B, n = 2100, 900, 70, 3
    scenes = [Scene(4000 + i, S, B, 5) for i in range(n)]
    raws = [sc.generate(0, L) for sc in scenes]
    tabs = [(_dev.to_device(sc.dark), _dev.to_device(sc.coeff)) for sc in scenes]
    g = _dev.to_device(np.ones(L, np.float32))
    gains, gconst = [g] * n, [1.0] * n
    eager = StripBatch(L, S, B, n)
    eager.enqueue(raws, tabs, gains, gconst)
    assert eager.verify(raws, tabs, gains) == []
    st, fl = eager.flags()
    assert (st == 0).all() and not any(needs_redo(f) or f & 4 for f in fl)
    gb = StripBatch(L, S, B, n)
    gb.enqueue(raws, tabs, gains, gconst)   # warm-up outside capture
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        gb.enqueue(raws, tabs, gains, gconst)
    gb.plan.scores.zero_()
    graph.replay()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(gb.plan.scores, eager.plan.scores)
    assert torch.equal(gb.plan.mask, eager.plan.mask)
    assert torch.equal(gb.plan.ds.sigma_inv, eager.plan.ds.sigma_inv)
    assert torch.equal(gb.plan.thr, eager.plan.thr)


def test_mixed_shapes_rejected(P):
    a = strips(P, 1)[0]
    b = strips(P, 1, L=64)[0]
    with pytest.raises(ValueError, match="same shape"):
        P.detect_strips([a, b])
