"""Parity at the BASELINE geometries, full size (the reference
pins its path end to end the same way, pkg/tests/test_acceptance.py:102-118).

  c4  one whole strip, 16384 x 900 x 70 (seed 4000), through detect_strips
  c3  the whole high-band cube, 8192 x 1024 x 270 (raww moments, score_tcw)
  c5  one N = 8 line block, 16384 x 2048 x 128, through the R-GLOBAL protocol
  c2  60 chunks of 249 x 900 x 70 through StreamingRX vs the oracle's StreamingStats
  (c1, 2048 x 900 x 70, is tests/test_gpu_parity.py::test_c1_full_size_vs_oracle)

Inputs come from the device generator (bit-identical to oracle/synth.py,
tests/test_gpu_parity.py::TestGenerator).  Tolerances are BASELINE's:
mu / Sigma 1e-5 normwise, scores 1e-4 per pixel, masks exact outside the
1e-4 band around the threshold, ridge equal.  Sigma^-1 is checked in two
parts: against the reference's algorithm on EXACT radiance
(oracle.compute_stats_exact) it must agree to 1e-8 — that is what the kernels
compute — and its distance to the f32-radiance reference must be the
reference's own f32 rounding effect (no more than 1.5x it, or under 1e-5).
Measured numbers go to gpurun_out/parity_geometry.jsonl when that exists.
"""

import json
import os
import time
from pathlib import Path

import numpy as np
import pytest

from oracle import skyrx_oracle as O
from oracle import synth as osynth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

STATS_RTOL = 1e-5
SCORE_RTOL = 1e-4
MASK_BAND = 1e-4
INV_EXACT_RTOL = 1e-8
LOG = Path(__file__).resolve().parent.parent / "gpurun_out" / "parity_geometry.jsonl"


@pytest.fixture(scope="module")
def P():
    import paper_2602_13509_b200 as P
    from paper_2602_13509_b200 import build

    build.build()
    return P


def nw(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def record(name, **kw):
    if LOG.parent.is_dir():
        with open(LOG, "a") as fh:
            fh.write(json.dumps({"case": name, **kw}) + "\n")


def check(name, stats, scores, mask, threshold, raw, t, gains=None, exact=True):
    """Everything BASELINE asks of one background + its scores and mask."""
    t0 = time.perf_counter()
    gains = np.ones(raw.shape[0]) if gains is None else gains
    want_stats, want_sc, want_mask = O.detect(raw, t.dark, t.coeff, gains)
    out = {"pixels": int(want_sc.size),
           "mu_rel": nw(stats.mu, want_stats.mu), "sigma_rel": nw(stats.sigma, want_stats.sigma),
           "sigma_inv_rel": nw(stats.sigma_inv, want_stats.sigma_inv)}
    assert out["mu_rel"] < STATS_RTOL and out["sigma_rel"] < STATS_RTOL, out
    assert stats.ridge_used == want_stats.ridge_used
    if exact:
        ex = O.compute_stats_exact(raw, t.dark, t.coeff, gains)
        out["sigma_inv_rel_vs_exact"] = nw(stats.sigma_inv, ex.sigma_inv)
        out["reference_f32_rounding"] = nw(want_stats.sigma_inv, ex.sigma_inv)
        assert out["sigma_inv_rel_vs_exact"] < INV_EXACT_RTOL, out
        assert (out["sigma_inv_rel"] < STATS_RTOL
                or out["sigma_inv_rel"] <= 1.5 * out["reference_f32_rounding"]), out
    rel = np.abs(scores - want_sc) / np.maximum(want_sc, 1e-12)
    out["score_max_rel"] = float(rel.max())
    assert out["score_max_rel"] < SCORE_RTOL, out
    thr = O.topk_threshold(want_sc)
    out["threshold_rel"] = abs(threshold - thr) / abs(thr)
    differ = mask != want_mask
    near = np.abs(want_sc - thr) <= MASK_BAND * abs(thr)
    out["mask_differ"] = int(differ.sum())
    out["mask_differ_outside_band"] = int((differ & ~near).sum())
    assert out["mask_differ_outside_band"] == 0, out
    out["oracle_s"] = time.perf_counter() - t0
    record(name, **out)
    return out


def device_raw(cfg, seed, line0=0, lines=None):
    from paper_2602_13509_b200.synth import Scene

    sc = Scene(seed, cfg["samples"], cfg["bands"], cfg["components"])
    return sc, sc.generate(line0, cfg["lines"] if lines is None else lines)


def test_c4_full_strip(P):
    """One whole c4 strip through the multi-strip API (StripBatch: the batched
    moments/finalize/score plan bench.py times), against the oracle."""
    c = osynth.CONFIGS["c4"]
    sc, rv = device_raw(c, c["seed"])
    raw = P.RawCube(rv, np.linspace(400, 1000, c["bands"]),
                    gains=np.ones(c["lines"], np.float32))
    res = P.detect_strips([(raw, P.CalibrationTables(sc.dark, sc.coeff))], host=True)
    det = res.local[0]
    check("c4_strip", det.stats, det.scores, det.mask, det.threshold, rv.cpu().numpy(), sc)


def test_c3_full_cube(P):
    """8192 x 1024 x 270: raw-byte wide moments (raww) + score_tcw at full size."""
    c = osynth.CONFIGS["c3"]
    sc, rv = device_raw(c, c["seed"])
    L, S, B = c["lines"], c["samples"], c["bands"]
    plan = P.DetectPlan(L, S, B)
    assert plan.tcw and plan.raw_stats
    raw = P.RawCube(rv, np.linspace(400, 1000, B), gains=np.ones(L, np.float32))
    det = P.detect(raw, P.CalibrationTables(sc.dark, sc.coeff), plan=plan, device=False)
    fl = int(plan.ds.flags[0].item())
    assert not fl & (2 | 4 | 16 | 32), fl   # the fast kernels applied
    check("c3_cube", det.stats, det.scores, det.mask, det.threshold, rv.cpu().numpy(), sc)


def test_c5_line_block(P):
    """One line block of the c5 mosaic at N = 8 (16384 of 131072 lines, block 3)
    through the R-GLOBAL protocol as a one-rank job (its own background)."""
    from paper_2602_13509_b200.distributed import GlobalRX

    c = osynth.CONFIGS["c5"]
    per = c["lines"] // 8
    sc, rv = device_raw(c, c["seed"], 3 * per, per)
    S, B = c["samples"], c["bands"]
    g = GlobalRX(per, S, B, P.CalibrationTables(sc.dark, sc.coeff), n_total=per * S)
    assert g.ops.plan.tcs
    det = g.detect(rv)
    fl = int(g.ops.plan.ds.flags[0].item())
    assert not fl & (2 | 4 | 16 | 32), fl
    check("c5_block", det.stats, det.scores.cpu().numpy(), det.mask.cpu().numpy(),
          det.threshold, rv.cpu().numpy(), sc)


def test_c2_sixty_chunks(P):
    """The full c2 stream: 60 chunks of 249 lines, forgetting 0.99, every chunk
    against the oracle's StreamingStats (stats, scores, mask)."""
    from paper_2602_13509_b200.stream import StreamingRX

    c = osynth.CONFIGS["c2"]
    L, S, B = c["chunk_lines"], c["samples"], c["bands"]
    nch = c["lines"] // L
    assert nch == 60
    sc, rv = device_raw(c, c["seed"], 0, L * nch)
    raw = rv.cpu().numpy()
    srx = StreamingRX(P.CalibrationTables(sc.dark, sc.coeff), L, c["forget"])
    ost = O.StreamingStats(B, c["forget"])
    worst = {"mu_rel": 0.0, "sigma_rel": 0.0, "sigma_inv_rel": 0.0, "score_max_rel": 0.0,
             "mask_differ": 0, "mask_differ_outside_band": 0}
    for i in range(nch):
        chunk = raw[i * L:(i + 1) * L]
        res = srx.update(rv[i * L:(i + 1) * L], with_stats=True)
        rad = O.apply_calibration(chunk, sc.dark, sc.coeff, np.ones(L))
        want = ost.update(rad)
        scores = O.rx_scores(rad, want)
        mask = O.topk_mask(scores)
        got_sc = res.scores.cpu().numpy()
        got_mask = res.mask.cpu().numpy()
        m = {"mu_rel": nw(res.stats.mu, want.mu), "sigma_rel": nw(res.stats.sigma, want.sigma),
             "sigma_inv_rel": nw(res.stats.sigma_inv, want.sigma_inv)}
        assert m["mu_rel"] < STATS_RTOL and m["sigma_rel"] < STATS_RTOL, (i, m)
        assert res.stats.ridge_used == want.ridge_used
        rel = np.abs(got_sc - scores) / np.maximum(scores, 1e-12)
        m["score_max_rel"] = float(rel.max())
        assert m["score_max_rel"] < SCORE_RTOL, (i, m)
        thr = O.topk_threshold(scores)
        differ = got_mask != mask
        near = np.abs(scores - thr) <= MASK_BAND * abs(thr)
        m["mask_differ"] = int(differ.sum())
        m["mask_differ_outside_band"] = int((differ & ~near).sum())
        assert m["mask_differ_outside_band"] == 0, (i, m)
        for key, v in m.items():
            worst[key] = max(worst[key], v) if "mask" not in key else worst[key] + v
    record("c2_stream_60", chunks=nch, **worst)
