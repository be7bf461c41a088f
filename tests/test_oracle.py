"""Pin the CPU oracle (oracle/skyrx_oracle.py) to the reference's own outputs.

Every fixture in tests/golden was produced by the real `skyrx` package
(tests/golden/make_golden.py).  These tests run on CPU.
"""

import numpy as np
import pytest

from conftest import case_names
from oracle import skyrx_oracle as O
from oracle import synth


class TestCalibrationOracle:
    def test_random_tables_bit_exact(self, golden):
        g = golden["calibrate"]
        out = O.apply_calibration(g["rand/raw"], g["rand/dark"], g["rand/coeff"], g["rand/gains"])
        assert out.dtype == np.float32
        assert np.array_equal(out.view(np.uint32), g["rand/out"].view(np.uint32))

    def test_by_definition(self, golden):
        assert (golden["calibrate"]["bydef/out"] == 45.0).all()

    def test_synth_cube_bit_exact(self, golden):
        g = golden["calibrate"]
        t = synth.make_tables(11, 96, 70)
        out = O.apply_calibration(g["synth/raw"], t.dark, t.coeff, g["synth/gains"])
        assert np.array_equal(out.view(np.uint32), g["synth/out"].view(np.uint32))

    @pytest.mark.parametrize("name", ["b300", "b44", "b340f8"])
    def test_fused_bin_rgb_bit_exact(self, golden, name):
        g = golden["calibrate"]
        out, centers, rgb = O.calibrate_bin_rgb(
            g[f"{name}/raw"], g[f"{name}/wl"], g[f"{name}/dark"], g[f"{name}/coeff"],
            g[f"{name}/gains"], factor=int(g[f"{name}/factor"]))
        assert np.array_equal(out.view(np.uint32), g[f"{name}/out"].view(np.uint32))
        assert np.array_equal(centers, g[f"{name}/centers"])
        assert np.array_equal(rgb.view(np.uint32), g[f"{name}/rgb"].view(np.uint32))

    @pytest.mark.parametrize("name", ["b300", "b44", "b340f8"])
    def test_sequential_band_sum_order(self, golden, name):
        # the CUDA binning kernel sums each group left to right; check that this is
        # exactly what the reference computes
        g = golden["calibrate"]
        f = int(g[f"{name}/factor"])
        rad = O.apply_calibration(g[f"{name}/raw"], g[f"{name}/dark"], g[f"{name}/coeff"],
                                  g[f"{name}/gains"])
        keep = O.keep_bands(g[f"{name}/wl"])
        x = rad[:, :, keep]
        x = x.reshape(x.shape[0], x.shape[1], -1, f)
        assert np.array_equal(O.sequential_sum_f32(x).view(np.uint32),
                              g[f"{name}/out"].view(np.uint32))

    def test_errors(self):
        with pytest.raises(ValueError, match="invalid tables"):
            O.apply_calibration(np.zeros((2, 3, 24), np.uint16), np.zeros((3, 23)),
                                np.ones((3, 23)), [1, 1])
        with pytest.raises(ValueError, match="every line gain must be positive"):
            O.apply_calibration(np.zeros((2, 3, 4), np.uint16), np.zeros((3, 4)),
                                np.ones((3, 4)), [1, 0])
        with pytest.raises(ValueError, match="divisible"):
            O.calibrate_bin_rgb(np.zeros((1, 2, 7), np.uint16), np.linspace(400, 1000, 7),
                                np.zeros((2, 7)), np.ones((2, 7)), [1.0], factor=4)

    def test_poisoned_gain_goes_non_finite(self):
        # test_pipeline.py:84-102: gain 1e-40 is an f32 subnormal -> inf radiance
        raw = np.full((2, 2, 3), 500, np.uint16)
        out = O.apply_calibration(raw, np.zeros((2, 3)), np.ones((2, 3)), [1.0, 1e-40])
        assert np.isinf(out[1]).all()
        with pytest.raises(ValueError, match="non-finite"):
            O.compute_stats(out)


class TestStatsOracle:
    def test_every_stats_case(self, golden):
        g = golden["stats"]
        for name in case_names(g, "mu"):
            st = O.compute_stats(g[f"{name}/values"])
            assert np.allclose(st.mu, g[f"{name}/mu"], rtol=1e-12, atol=1e-12), name
            assert np.allclose(st.sigma, g[f"{name}/sigma"], rtol=1e-10, atol=1e-12), name
            assert st.ridge_used == float(g[f"{name}/ridge"]), name
            assert np.allclose(st.chol_lower, g[f"{name}/chol"], rtol=1e-9, atol=1e-12), name
            sc = O.rx_scores(g[f"{name}/values"], st)
            want = g[f"{name}/scores"]
            rel = np.abs(sc - want) / np.maximum(np.abs(want), 1e-12)
            assert (rel < 1e-6).all() or np.array_equal(sc, want), name

    def test_degenerate_cases(self, golden):
        g = golden["stats"]
        assert float(g["ident/ridge"]) > 0 and (g["ident/scores"] == 0).all()
        assert float(g["rank1/ridge"]) > 0
        assert g["mean0/scores"][1, 0] == 0.0 and g["mean0/scores"][1, 1] == 0.0
        assert g["hand1/scores"][1, 1] == pytest.approx(2.25, rel=1e-6)

    def test_errors(self, rng):
        with pytest.raises(ValueError, match="insufficient"):
            O.compute_stats(rng.random((1, 3, 4), dtype=np.float32))
        with pytest.raises(ValueError, match="bands"):
            O.rx_scores(rng.random((4, 4, 5), dtype=np.float32),
                        O.compute_stats(rng.random((4, 4, 3), dtype=np.float32)))

    def test_mahalanobis_slot(self, golden):
        a = golden["accel"]
        d = O.mahalanobis_sq(a["px"], a["mu"], a["chol"], chunk=997)
        assert np.allclose(d, a["numpy"], rtol=1e-12, atol=0)
        assert np.allclose(d, a["numba"], rtol=1e-9, atol=0)

    def test_synth_threshold_mask(self, golden):
        g = golden["stats"]
        for name in ("synth70", "synth128"):
            norm = O.normalize_scores(g[f"{name}/scores"])
            assert np.array_equal(norm, g[f"{name}/norm"])
            assert np.array_equal(O.threshold_scores(norm, 0.11), g[f"{name}/mask_t"])


class TestNormalizeOracle:
    def test_cases(self, golden):
        g = golden["normalize"]
        assert np.array_equal(O.normalize_scores(g["rand/values"]), g["rand/norm"])
        assert np.array_equal(O.threshold_scores(g["rand/norm"], 0.37), g["rand/mask037"])
        assert np.array_equal(O.threshold_scores(g["small/norm"], 1.0), g["small/mask1"])
        assert np.array_equal(O.threshold_scores(g["small/norm"], 0.0), g["small/mask0"])
        t = float(g["edge/t"])
        assert np.array_equal(O.threshold_scores(g["edge/values"], t), g["edge/mask"])
        assert not g["edge/mask"][0, 0]   # NEP 50: t rounds to f32 before the compare
        assert float(g["edge/values"][0, 0]) > t

    def test_threshold_range(self):
        for bad in (-0.1, 1.5):
            with pytest.raises(ValueError, match="threshold"):
                O.threshold_scores(np.zeros((2, 2), np.float32), bad)

    def test_transmit_domain(self):
        v = np.array([[0.0, 1.0], [4.0, 16.0]])
        assert np.allclose(O.transmit_domain(v, 16.0), [[0, 0.25], [0.5, 1.0]])
        assert (O.transmit_domain(v, 0.0) == 0).all()


class TestNewRows:
    """R-TOPK / R-GLOBAL / R-STREAM definitions (no reference implementation)."""

    def test_topk_definition(self, rng):
        s = rng.random(10_000).astype(np.float32)
        k = O.topk_count(s.size)
        assert k == 10
        m = O.topk_mask(s)
        assert m.sum() == k
        assert s[m].min() > s[~m].max()

    def test_topk_ties_and_small(self):
        s = np.array([1, 2, 2, 2, 0], np.float32)
        assert O.topk_count(5) == 1
        assert O.topk_mask(s).sum() == 0           # threshold = 2 ties with the top
        assert O.topk_mask(np.ones(1, np.float32)).all()   # k >= N selects everything

    def test_global_combine_equals_single(self, rng):
        x = rng.normal(100, 5, (40, 30, 6)).astype(np.float32)
        ref = O.compute_stats(x)
        c = x[0, 0].astype(np.float64)
        parts = [O.moments(x[i:i + 10], c) for i in range(0, 40, 10)]
        st = O.finalize_moments(*O.combine_moments(parts), c)
        assert np.allclose(st.mu, ref.mu, rtol=1e-12)
        assert np.allclose(st.sigma, ref.sigma, rtol=1e-9)
        assert st.ridge_used == ref.ridge_used

    def test_stream_chunk0_equals_compute_stats(self, rng):
        x = rng.normal(50, 3, (20, 16, 5)).astype(np.float32)
        ss = O.StreamingStats(5, 0.99)
        st = ss.update(x)
        ref = O.compute_stats(x)
        assert np.allclose(st.mu, ref.mu, rtol=1e-12)
        assert np.allclose(st.sigma, ref.sigma, rtol=1e-9)
        st2 = ss.update(x + 1)
        assert ss.n == pytest.approx(0.99 * 320 + 320)
        assert not np.allclose(st2.mu, st.mu)


class TestGenerator:
    def test_deterministic_and_blockwise(self):
        t = synth.make_tables(3, 40, 12)
        a = synth.generate_lines(t, 0, 20)
        b = np.concatenate([synth.generate_lines(t, 0, 7), synth.generate_lines(t, 7, 13)])
        assert np.array_equal(a, b)
        assert a.dtype == np.uint16 and a.max() <= 4095

    def test_anomaly_fraction(self):
        t = synth.make_tables(1, 900, 70)
        frac = synth.anomaly_mask(t, 0, 2048).mean()
        assert 0.0007 < frac < 0.0014

    def test_golden_inputs_regenerate(self, golden):
        t = synth.make_tables(21, 64, 70)
        assert np.array_equal(synth.generate_lines(t, 0, 48), golden["stats"]["synth70/raw"])


# ----------------------------------------------------------------------------- link payload
def test_link_payload_matches_reference(golden):
    g = golden["datalink"]
    assert np.array_equal(O.pack_rgb565(g["row/rgb"], 40.0, 37.5, 12.25), g["row/rgb565"])
    assert np.array_equal(O.encode_scores_half(g["row/scores"], 500.0), g["row/half"])
    assert np.array_equal(O.encode_scores_half(g["row/scores"], 0.0), g["row/half_zero_max"])
    assert np.array_equal(O.pack_rgb565(g["row/rgb"], 0.0, 37.5, -1.0), g["row/rgb565_zero_max"])


def test_packetize_cube_matches_reference(golden):
    g = golden["datalink"]
    lines = g["cube/rgb"].shape[0]
    metas = []
    for i in range(lines):  # tests/golden/make_golden.py metas()
        t = 1_600_000_000_000_000 + i * 4016
        metas.append((t, (t - 1000, 35.0, -90.0, 40.0, 0.0, 0.0, 0.0),
                      (t + 4000, 35.0, -90.0, 40.0, 0.0, 0.0, 0.0)))
    pk = O.packetize_cube(7, g["cube/rgb"], g["cube/scores"], metas)
    assert all(len(p) == 3728 for p in pk)
    assert np.array_equal(np.frombuffer(b"".join(pk), np.uint8), g["cube/packets"])


def test_gf_oracle_matches_reference(golden):
    g = golden["fec"]
    assert np.array_equal(O.GF_LOG_T, g["gf_log"]) and np.array_equal(O.GF_EXP_T, g["gf_exp"])
    assert np.array_equal(O.gf256_matmul(g["mm/mat"], g["mm/data"]), g["mm/out"])
    assert np.array_equal(O.gf_mat_inv(g["inv/m"]), g["inv/minv"])
    for k, p in ((50, 25), (4, 3), (1, 0), (200, 56)):
        assert np.array_equal(O.encoding_matrix(k, k + p), g[f"matrix_{k}_{p}"]), (k, p)


def test_rs_oracle_matches_reference(golden):
    g = golden["fec"]
    m = g["matrix_50_25"]
    coded = [r.tobytes() for r in g["enc/coded"]]
    assert O.rs_encode(m, 50, coded[:50]) == coded[50:]
    c = 0
    while f"dec{c}/keep" in g:
        out, (rec, recov, miss) = O.rs_decode(m, 50, [(int(i), coded[i]) for i in g[f"dec{c}/keep"]])
        assert sorted(out) == g[f"dec{c}/slots"].tolist()
        assert b"".join(out[i] for i in sorted(out)) == g[f"dec{c}/data"].tobytes()
        assert [len(rec), len(recov), len(miss)] == g[f"dec{c}/report"].tolist()
        assert list(recov) == g[f"dec{c}/recovered"].tolist()
        assert list(miss) == g[f"dec{c}/missing"].tolist()
        c += 1
    assert c == 10
    pk = g["frames/packets"].reshape(100, -1)
    fr = b"".join(O.frames_for_cube(3, [r.tobytes() for r in pk], matrix=m))
    assert fr == g["frames/frames"].tobytes()
