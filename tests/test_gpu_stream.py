"""R-STREAM (BASELINE config 2) on the GPU vs the CPU oracle's StreamingStats.

Per chunk: the device background (f64 moments folded with forgetting 0.99,
finalized on device) against oracle/skyrx_oracle.py StreamingStats.update,
scores and top-0.1% masks against the oracle scored with those stats.
Tolerances as tests/test_gpu_parity.py (stats 1e-5, Sigma^-1 1e-3 derived,
scores 1e-4 per pixel, masks exact outside the 1e-4 threshold band).
"""

import numpy as np
import pytest

from oracle import skyrx_oracle as O
from oracle import synth as osynth

pytestmark = pytest.mark.gpu

STATS_RTOL = 1e-5
INV_RTOL = 1e-5
SCORE_RTOL = 1e-4
MASK_BAND = 1e-4


@pytest.fixture(scope="module")
def P():
    import paper_2602_13509_b200 as P
    from paper_2602_13509_b200 import build

    build.build()
    return P


def normwise(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300)


def oracle_stream(raw_chunks, t, forget):
    st = O.StreamingStats(t.dark.shape[1], forget)
    out = []
    for raw in raw_chunks:
        rad = O.apply_calibration(raw, t.dark, t.coeff, np.ones(raw.shape[0]))
        stats = st.update(rad)
        scores = O.rx_scores(rad, stats)
        out.append((stats, scores, O.topk_mask(scores)))
    return out


def check_chunk(res, want):
    stats, scores, mask = want
    assert normwise(res.stats.mu, stats.mu) < STATS_RTOL
    assert normwise(res.stats.sigma, stats.sigma) < STATS_RTOL
    assert normwise(res.stats.sigma_inv, stats.sigma_inv) < INV_RTOL
    assert res.stats.ridge_used == stats.ridge_used
    rel = np.abs(res.scores - scores) / np.maximum(scores, 1e-12)
    assert rel.max() < SCORE_RTOL, rel.max()
    thr = O.topk_threshold(scores)
    assert res.threshold == pytest.approx(thr, rel=SCORE_RTOL)
    near = np.abs(scores - thr) <= MASK_BAND * abs(thr)
    assert not ((res.mask != mask) & ~near).any()


@pytest.mark.parametrize("S,B,chunk,nchunks", [(96, 70, 249, 6), (64, 48, 100, 4), (40, 16, 37, 5)])
def test_stream_matches_oracle(P, S, B, chunk, nchunks):
    from paper_2602_13509_b200.stream import StreamingRX

    t = osynth.make_tables(2, S, B, 5)
    raws = [osynth.generate_lines(t, i * chunk, chunk) for i in range(nchunks)]
    want = oracle_stream(raws, t, 0.99)
    srx = StreamingRX(P.CalibrationTables(t.dark, t.coeff), chunk_lines=chunk, forget=0.99)
    for raw, w in zip(raws, want):
        check_chunk(srx.update(raw, with_stats=True), w)


def test_graph_replay_bit_identical_to_eager(P):
    from paper_2602_13509_b200.stream import StreamingRX

    t = osynth.make_tables(2, 96, 70, 5)
    raws = [osynth.generate_lines(t, i * 249, 249) for i in range(4)]
    tabs = P.CalibrationTables(t.dark, t.coeff)
    a = StreamingRX(tabs, 249, use_graph=True)
    b = StreamingRX(tabs, 249, use_graph=False)
    for raw in raws:
        ra, rb = a.update(raw, with_stats=True), b.update(raw, with_stats=True)
        assert np.array_equal(ra.scores.view(np.uint32), rb.scores.view(np.uint32))
        assert np.array_equal(ra.mask, rb.mask)
        assert np.array_equal(ra.stats.sigma_inv, rb.stats.sigma_inv)
    assert a.graph is not None and b.graph is None


def test_forget_one_equals_batch_fit(P):
    """lambda = 1: the folded state is the moments of all chunks so far."""
    from paper_2602_13509_b200.stream import StreamingRX

    t = osynth.make_tables(7, 64, 70, 5)
    raws = [osynth.generate_lines(t, i * 120, 120) for i in range(3)]
    srx = StreamingRX(P.CalibrationTables(t.dark, t.coeff), 120, forget=1.0)
    for raw in raws:
        res = srx.update(raw, with_stats=True)
    allraw = np.concatenate(raws)
    rad = O.apply_calibration(allraw, t.dark, t.coeff, np.ones(allraw.shape[0]))
    want = O.compute_stats(rad)
    # the raw-byte moments calibrate each integer Gram exactly in f64, the oracle
    # sums f32-rounded radiance (calibrate.py:98-101): they agree to that rounding
    assert normwise(res.stats.mu, want.mu) < 1e-8
    assert normwise(res.stats.sigma, want.sigma) < 1e-7


def test_clamped_chunk_falls_back_to_f64(P):
    """A chunk with values below dark cannot use the raw-byte moments: the chunk is
    redone in f64 from the pre-chunk state and still matches the oracle."""
    from paper_2602_13509_b200.stream import StreamingRX

    t = osynth.make_tables(2, 96, 70, 5)
    raws = [osynth.generate_lines(t, i * 249, 249).copy() for i in range(4)]
    raws[2][10, 20, 5] = 0  # below dark: clamps to 0 radiance
    want = oracle_stream(raws, t, 0.99)
    srx = StreamingRX(P.CalibrationTables(t.dark, t.coeff), 249)
    for raw, w in zip(raws, want):
        check_chunk(srx.update(raw, with_stats=True), w)


def test_device_chunks_stay_on_device(P):
    import torch
    from paper_2602_13509_b200.stream import StreamingRX

    t = osynth.make_tables(2, 96, 70, 5)
    raw = osynth.generate_lines(t, 0, 249)
    srx = StreamingRX(P.CalibrationTables(t.dark, t.coeff), 249)
    res = srx.update(torch.from_numpy(raw).cuda())
    assert isinstance(res.scores, torch.Tensor) and res.scores.is_cuda
    host = StreamingRX(P.CalibrationTables(t.dark, t.coeff), 249).update(raw)
    assert np.array_equal(res.scores.cpu().numpy(), host.scores)


def test_errors(P):
    from paper_2602_13509_b200.stream import StreamingRX

    t = osynth.make_tables(2, 32, 16, 3)
    srx = StreamingRX(P.CalibrationTables(t.dark, t.coeff), 10)
    with pytest.raises(ValueError, match="geometry"):
        srx.update(np.zeros((11, 32, 16), np.uint16))
    with pytest.raises(ValueError, match="forget"):
        StreamingRX(P.CalibrationTables(t.dark, t.coeff), 10, forget=1.5)
