"""CUDA path vs the reference's golden outputs and the pinned CPU oracle.

All tests need a B200 (`-m gpu`); they call the hand-written kernels through
the C ABI (paper_2602_13509_b200._lib) and compare with:
  * tests/golden/*.npz — produced by the real reference package;
  * oracle/ — the CPU restatement pinned to those goldens (tests/test_oracle.py).
Tolerances: calibration bit-exact; precise-mode stats/scores at the
reference's own test tolerances; fast mode at BASELINE's 1e-5 (stats,
normwise) and 1e-4 (scores, per pixel); masks bit-exact except pixels whose
reference score lies within 1e-4 relative of the reference threshold.
"""

import numpy as np
import pytest

from conftest import case_names
from oracle import skyrx_oracle as O
from oracle import synth as osynth

pytestmark = pytest.mark.gpu

STATS_RTOL_FAST = 1e-5      # BASELINE.json north_star: stats within 1e-5 relative
INV_RTOL_FAST = 1e-5        # ... Sigma^-1 included (measured <= 2.1e-8 at every BASELINE
                            # geometry, profiles/r02_parity_geometry.jsonl)
SCORE_RTOL_FAST = 1e-4      # scores within 1e-4 relative
MASK_BAND = 1e-4            # mask exemption band around the threshold


@pytest.fixture(scope="module")
def P():
    import paper_2602_13509_b200 as P
    from paper_2602_13509_b200 import build

    build.build()
    return P


def raw_cube(P, values, gains=None, wl=None):
    values = np.asarray(values, np.uint16)
    if gains is None:
        gains = np.ones(values.shape[0])
    if wl is None:
        wl = np.linspace(400, 1000, values.shape[2])
    return P.RawCube(values, wl, P.cube.line_meta_for(gains))


def rad_cube(P, values):
    values = np.asarray(values, np.float32)
    return P.RadianceCube(values, np.linspace(400, 1000, values.shape[2]),
                          P.cube.line_meta_for([2.0] * values.shape[0]))


def bits(a):
    return np.asarray(a, np.float32).view(np.uint32)


def normwise(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300)


# ----------------------------------------------------------------------------- generator
class TestGenerator:
    @pytest.mark.parametrize("args,line0,n", [((1, 900, 70, 5), 0, 40), ((3, 64, 270, 8), 500, 9),
                                              ((5, 40, 128, 5), 131000, 12),
                                              ((4007, 900, 70, 5), 16000, 16)])
    def test_device_generator_bit_identical(self, P, args, line0, n):
        from paper_2602_13509_b200.synth import Scene

        dev = Scene(*args).generate(line0, n).cpu().numpy()
        host = osynth.generate_lines(osynth.make_tables(*args), line0, n)
        assert np.array_equal(dev, host)


# ----------------------------------------------------------------------------- calibration
class TestCalibration:
    def test_random_tables_bit_exact(self, P, golden):
        g = golden["calibrate"]
        raw = raw_cube(P, g["rand/raw"], g["rand/gains"])
        out = P.apply_calibration(raw, P.CalibrationTables(g["rand/dark"], g["rand/coeff"]))
        assert np.array_equal(bits(out.values), bits(g["rand/out"]))

    def test_synth_with_line_gains_bit_exact(self, P, golden):
        g = golden["calibrate"]
        t = osynth.make_tables(11, 96, 70)
        out = P.apply_calibration(raw_cube(P, g["synth/raw"], g["synth/gains"]),
                                  P.CalibrationTables(t.dark, t.coeff))
        assert np.array_equal(bits(out.values), bits(g["synth/out"]))

    def test_by_definition_and_clamp(self, P):
        raw = raw_cube(P, np.full((1, 1, 24), 100), [4.0])
        t = P.CalibrationTables(np.full((1, 24), 10.0), np.full((1, 24), 2.0))
        assert (P.apply_calibration(raw, t).values == 45.0).all()
        raw = raw_cube(P, np.full((1, 1, 24), 5))
        t = P.CalibrationTables(np.full((1, 24), 10.0), np.ones((1, 24)))
        assert (P.apply_calibration(raw, t).values == 0).all()

    def test_unaligned_shapes(self, P, rng):
        # odd S*B takes the scalar kernel; results must still be bit-exact
        raw = rng.integers(0, 4096, (5, 7, 13)).astype(np.uint16)
        dark = rng.uniform(0, 50, (7, 13)).astype(np.float32)
        coeff = rng.uniform(0.5, 2, (7, 13)).astype(np.float32)
        gains = rng.uniform(1, 8, 5)
        out = P.apply_calibration(raw_cube(P, raw, gains), P.CalibrationTables(dark, coeff))
        want = O.apply_calibration(raw, dark, coeff, gains)
        assert np.array_equal(bits(out.values), bits(want))

    def test_poisoned_gain_is_inf_then_nonfinite(self, P):
        # test_pipeline.py:84-102: 1e-40 is subnormal in f32 and must not flush
        raw = raw_cube(P, np.full((2, 2, 3), 500), [1.0, 1e-40])
        t = P.CalibrationTables(np.zeros((2, 3)), np.ones((2, 3)))
        out = P.apply_calibration(raw, t)
        assert np.isinf(out.values[1]).all() and np.isfinite(out.values[0]).all()
        with pytest.raises(ValueError, match="non-finite"):
            P.compute_stats(out)
        with pytest.raises(ValueError, match="non-finite"):
            P.compute_stats(out, mode="fast")
        with pytest.raises(ValueError, match="non-finite"):
            P.detect(raw, t)

    def test_nan_dark_is_nonfinite(self, P):
        # np.maximum keeps NaN (calibrate.py:99), so a NaN dark entry makes that
        # radiance column NaN and the fit raises rx.py:53-54's error, on every path
        L, S, B = 300, 900, 70
        t = osynth.make_tables(46, S, B, 5)
        raw = osynth.generate_lines(t, 0, L)
        dark = t.dark.copy()
        dark[17, 3] = np.nan
        tab = P.CalibrationTables(dark, t.coeff)
        out = P.apply_calibration(raw_cube(P, raw), tab).values
        want = O.apply_calibration(raw, dark, t.coeff, np.ones(L))
        assert np.array_equal(np.isnan(out), np.isnan(want)) and np.isnan(want).sum() == L
        ok = ~np.isnan(want)
        assert np.array_equal(bits(out[ok]), bits(want[ok]))
        with pytest.raises(ValueError, match="non-finite"):
            P.detect(raw_cube(P, raw), tab)
        with pytest.raises(ValueError, match="non-finite"):
            P.compute_stats(P.RadianceCube(out, np.linspace(400, 1000, B),
                                           P.cube.line_meta_for([1.0] * L)))

    @pytest.mark.parametrize("name", ["b300", "b44", "b340f8"])
    def test_fused_bin_rgb_bit_exact(self, P, golden, name):
        g = golden["calibrate"]
        raw = raw_cube(P, g[f"{name}/raw"], g[f"{name}/gains"], g[f"{name}/wl"])
        cube, rgb = P.calibrate_bin_rgb(raw, P.CalibrationTables(g[f"{name}/dark"],
                                                                 g[f"{name}/coeff"]),
                                        factor=int(g[f"{name}/factor"]))
        assert np.array_equal(bits(cube.values), bits(g[f"{name}/out"]))
        assert np.array_equal(cube.wavelengths_nm, g[f"{name}/centers"])
        assert np.array_equal(bits(rgb), bits(g[f"{name}/rgb"]))

    @pytest.mark.parametrize("S", [900, 7])
    def test_fused_rgb_targets_sharing_a_band(self, P, rng, S):
        """Few output bands (the reference pipeline suite's 32 bands over -145..1545 nm ->
        3 binned bands at factor 4): RGB targets that pick the same band all get written
        (the tiled kernel once wrote one, leaving the other uninitialised)."""
        L, B = 100, 32
        wl = np.linspace(-145.45454407, 1545.45458984, B)
        t = osynth.make_tables(7, S, B)
        raw = rng.integers(80, 4000, size=(L, S, B), dtype=np.uint16)
        gains = 1.0 + 0.1 * rng.random(L)
        # 11 bands inside 400-1000 nm, binned by 11 -> one output band for all three targets
        cube, rgb = P.calibrate_bin_rgb(raw_cube(P, raw, gains, wl),
                                        P.CalibrationTables(t.dark, t.coeff), factor=11)
        out, centers, want_rgb = O.calibrate_bin_rgb(raw, wl, t.dark, t.coeff, gains, factor=11)
        idx = [O.band_nearest(centers, x) for x in O.RGB_TARGETS_NM]
        assert len(set(idx)) < 3  # the case under test
        assert np.array_equal(bits(cube.values), bits(out))
        assert np.array_equal(bits(rgb), bits(want_rgb))

    def test_composed_ops_match_fused(self, P, golden):
        g = golden["calibrate"]
        raw = raw_cube(P, g["b300/raw"], g["b300/gains"], g["b300/wl"])
        t = P.CalibrationTables(g["b300/dark"], g["b300/coeff"])
        composed = P.bin_bands(P.discard_oob_bands(P.apply_calibration(raw, t)), 4)
        assert composed.bands == 70
        assert np.array_equal(bits(composed.values), bits(g["b300/out"]))
        assert np.array_equal(bits(P.extract_rgb(composed)), bits(g["b300/rgb"]))

    def test_bin_all_ones_and_sum_preserved(self, P, rng):
        cube = rad_cube(P, np.ones((2, 3, 280), np.float32))
        assert (P.bin_bands(cube, 4).values == 4.0).all()
        vals = rng.integers(0, 256, (3, 4, 280)).astype(np.float32)
        out = P.bin_bands(rad_cube(P, vals), 4)
        assert np.sum(out.values, dtype=np.float64) == np.sum(vals, dtype=np.float64)

    def test_device_tensors_stay_on_device(self, P, golden):
        import torch

        g = golden["calibrate"]
        raw = P.RawCube(torch.from_numpy(g["rand/raw"]).cuda(), np.linspace(400, 1000, 24),
                        gains=torch.tensor(g["rand/gains"], dtype=torch.float32).cuda())
        out = P.apply_calibration(raw, P.CalibrationTables(g["rand/dark"], g["rand/coeff"]))
        assert isinstance(out.values, torch.Tensor) and out.values.is_cuda
        assert np.array_equal(bits(out.values.cpu().numpy()), bits(g["rand/out"]))


# ----------------------------------------------------------------------------- statistics
class TestStatsPrecise:
    def test_every_golden_case(self, P, golden):
        g = golden["stats"]
        for name in case_names(g, "mu"):
            st = P.compute_stats(rad_cube(P, g[f"{name}/values"]))
            assert np.allclose(st.mu, g[f"{name}/mu"], rtol=1e-12, atol=1e-9), name
            assert np.allclose(st.sigma, g[f"{name}/sigma"], rtol=1e-9, atol=1e-9), name
            assert st.ridge_used == float(g[f"{name}/ridge"]), name
            assert np.allclose(st.chol_lower, g[f"{name}/chol"], rtol=1e-8, atol=1e-9), name
            assert normwise(st.sigma_inv, g[f"{name}/sigma_inv"]) < 1e-8, name

    def test_every_golden_case_scores(self, P, golden):
        g = golden["stats"]
        for name in case_names(g, "mu"):
            cube = rad_cube(P, g[f"{name}/values"])
            sc = P.rx_scores(cube, P.compute_stats(cube)).values
            want = g[f"{name}/scores"]
            rel = np.abs(sc - want) / np.maximum(np.abs(want), 1e-12)
            assert (rel < 1e-6).all(), (name, rel.max())

    def test_degenerate(self, P):
        cube = rad_cube(P, np.full((4, 4, 3), 9.0))
        st = P.compute_stats(cube)
        assert (st.sigma == 0).all() and st.ridge_used > 0
        assert (P.rx_scores(cube, st).values == 0).all()
        base = np.arange(16, dtype=np.float32)
        cube = rad_cube(P, np.stack([base, 2 * base], axis=1).reshape(4, 4, 2))
        st = P.compute_stats(cube)
        assert st.ridge_used > 0 and np.isfinite(P.rx_scores(cube, st).values).all()

    def test_errors(self, P, rng):
        with pytest.raises(ValueError, match="insufficient"):
            P.compute_stats(rad_cube(P, rng.random((1, 3, 4), dtype=np.float32)))
        vals = np.ones((3, 3, 2), np.float32)
        vals[1, 1, 0] = np.inf
        with pytest.raises(ValueError, match="non-finite"):
            P.compute_stats(rad_cube(P, vals))
        a = rad_cube(P, rng.random((4, 4, 3), dtype=np.float32))
        b = rad_cube(P, rng.random((4, 4, 5), dtype=np.float32))
        with pytest.raises(ValueError, match="bands"):
            P.rx_scores(b, P.compute_stats(a))

    def test_permutation_invariance_rtol_1e9(self, P, rng):
        # test_rx.py:144-158 at the reference's own tolerance (precise mode)
        vals = rng.normal(10, 2, (6, 8, 3)).astype(np.float32)
        s1 = P.rx_scores(rad_cube(P, vals), P.compute_stats(rad_cube(P, vals))).values.ravel()
        perm = rng.permutation(48)
        sh = vals.reshape(-1, 3)[perm].reshape(6, 8, 3)
        s2 = P.rx_scores(rad_cube(P, sh), P.compute_stats(rad_cube(P, sh))).values.ravel()
        assert np.allclose(s2, s1[perm], rtol=1e-9, atol=1e-9)

    def test_large_band_counts(self, P):
        # B = 270 / 300 exercise the multi-part Gram and the global-memory Cholesky
        for b in (128, 270, 300):
            t = osynth.make_tables(77, 48, b, 8)
            raw = osynth.generate_lines(t, 0, 40)
            rad = O.apply_calibration(raw, t.dark, t.coeff, np.ones(40))
            want = O.compute_stats(rad)
            st = P.compute_stats(rad_cube(P, rad))
            assert normwise(st.sigma, want.sigma) < 1e-12, b
            assert st.ridge_used == want.ridge_used
            assert normwise(st.sigma_inv, want.sigma_inv) < 1e-6, b
            sc = P.rx_scores(rad_cube(P, rad), st).values
            ref = O.rx_scores(rad, want)
            assert (np.abs(sc - ref) / ref).max() < 1e-5, b


class TestAccelSlot:
    def test_matches_reference_numba(self, P, golden):
        from paper_2602_13509_b200 import _accel

        a = golden["accel"]
        d = _accel.mahalanobis_sq(a["px"], a["mu"], a["chol"])
        assert d.dtype == np.float64
        assert (np.abs(d - a["numba"]) / np.abs(a["numba"])).max() < 1e-9
        d64 = _accel.mahalanobis_sq(a["px"].astype(np.float64), a["mu"], a["chol"])
        assert (np.abs(d64 - a["numpy"]) / np.abs(a["numpy"])).max() < 1e-9


class TestFastMode:
    @pytest.mark.parametrize("name", ["synth70", "synth128", "normal", "acc0", "acc3"])
    def test_stats_and_scores_within_baseline_tolerance(self, P, golden, name):
        g = golden["stats"]
        cube = rad_cube(P, g[f"{name}/values"])
        st = P.compute_stats(cube, mode="fast")
        assert normwise(st.mu, g[f"{name}/mu"]) < STATS_RTOL_FAST
        assert normwise(st.sigma, g[f"{name}/sigma"]) < STATS_RTOL_FAST
        inv = normwise(st.sigma_inv, g[f"{name}/sigma_inv"])
        print(f"PARITY fast-mode {name} sigma_inv {inv:.3e}")
        assert inv < INV_RTOL_FAST, inv
        assert st.ridge_used == float(g[f"{name}/ridge"])
        sc = P.rx_scores(cube, st, mode="fast").values
        want = g[f"{name}/scores"]
        assert (np.abs(sc - want) / np.maximum(want, 1e-12)).max() < SCORE_RTOL_FAST

    @pytest.mark.parametrize("S,B,L", [(900, 70, 1000), (256, 48, 2048), (900, 72, 400)])
    def test_radiance_cube_moments_on_tensor_cores(self, P, monkeypatch, S, B, L):
        """compute_stats(RadianceCube, mode="fast") takes the quantised-digit tensor-core
        Gram (skyrx_stats_tc_f32) and meets the 1e-5 statistics tolerance; the paper's
        binned cube shape (1000 x 900 x 70) first."""
        from paper_2602_13509_b200 import _lib

        t = osynth.make_tables(51, S, B, 5)
        raw = osynth.generate_lines(t, 0, L)
        rad = O.apply_calibration(raw, t.dark, t.coeff, np.ones(L))
        calls = []
        real = _lib.call
        monkeypatch.setattr(_lib, "call", lambda name, *a: (calls.append(name), real(name, *a))[1])
        st = P.compute_stats(rad_cube(P, rad), mode="fast")
        assert "skyrx_stats_tc_f32" in calls
        want = O.compute_stats(rad)
        assert normwise(st.mu, want.mu) < STATS_RTOL_FAST
        assert normwise(st.sigma, want.sigma) < STATS_RTOL_FAST
        inv = normwise(st.sigma_inv, want.sigma_inv)
        print(f"PARITY tc-f32 moments {S}x{B}x{L} sigma_inv {inv:.3e}")
        assert inv < INV_RTOL_FAST, inv
        assert st.ridge_used == want.ridge_used

    def test_radiance_cube_nonfinite_on_tensor_cores(self, P):
        t = osynth.make_tables(52, 900, 70, 5)
        rad = O.apply_calibration(osynth.generate_lines(t, 0, 400), t.dark, t.coeff, np.ones(400))
        rad[123, 45, 6] = np.inf
        with pytest.raises(ValueError, match="non-finite"):
            P.compute_stats(rad_cube(P, rad), mode="fast")


# ----------------------------------------------------------------------------- normalise etc.
class TestNormalize:
    def test_golden(self, P, golden):
        g = golden["normalize"]
        n = P.normalize_scores(P.ScoreMap(g["rand/values"]))
        assert np.array_equal(bits(n.values), bits(g["rand/norm"]))
        assert np.array_equal(P.threshold_scores(n, 0.37), g["rand/mask037"])
        n = P.normalize_scores(P.ScoreMap(g["small/values"]))
        assert np.array_equal(P.threshold_scores(n, 1.0), g["small/mask1"])
        assert np.array_equal(P.threshold_scores(n, 0.0), g["small/mask0"])
        m = P.threshold_scores(P.ScoreMap(g["edge/values"]), float(g["edge/t"]))
        assert np.array_equal(m, g["edge/mask"])

    def test_zero_map_and_synth(self, P, golden):
        z = P.ScoreMap(np.zeros((2, 2)))
        assert (P.normalize_scores(z).values == 0).all()
        g = golden["stats"]
        n = P.normalize_scores(P.ScoreMap(g["synth70/scores"]))
        assert np.array_equal(bits(n.values), bits(g["synth70/norm"]))
        assert np.array_equal(P.threshold_scores(n, 0.11), g["synth70/mask_t"])

    def test_transmit_domain(self, P, rng):
        v = rng.random((7, 9)).astype(np.float32) * 20
        got = P.transmit_domain(v, 17.5)
        assert got.dtype == np.float64
        assert np.array_equal(got, O.transmit_domain(v, 17.5))
        assert (P.transmit_domain(v, 0.0) == 0).all()


class TestTopK:
    @pytest.mark.parametrize("n,k", [(10_000, None), (1_843_200, None), (5, 1), (1, None),
                                     (1000, 999), (1000, 1000), (0, None)])
    def test_matches_oracle(self, P, rng, n, k):
        v = (rng.random(n) * rng.choice([1, 10, 1e4], n)).astype(np.float32)
        got = P.topk_mask(v, k)
        assert np.array_equal(got, O.topk_mask(v, k))

    @pytest.mark.parametrize("n", [3, 8, 4099])
    def test_select_all_includes_inf_and_nan(self, P, n):
        # k >= n: the oracle returns np.ones, so -inf and NaN scores are selected too
        v = np.arange(n, dtype=np.float32)
        v[0], v[-1] = -np.inf, np.nan
        assert P.topk_mask(v, n).all() and O.topk_mask(v, n).all()
        assert P.topk_mask(v, n + 5).all()

    def test_ties(self, P):
        v = np.array([1, 2, 2, 2, 0], np.float32)
        assert np.array_equal(P.topk_mask(v), O.topk_mask(v))
        v = np.full(5000, 3.0, np.float32)
        assert not P.topk_mask(v).any()

    @pytest.mark.parametrize("n,cap", [(100_003, 0), (100_003, 7), (1_843_201, None),
                                       (4099, None), (3, None)])
    def test_one_pass_mask_equals_threshold_then_mask(self, P, rng, n, cap):
        """skyrx_topk_mask (candidates, or the in-bin rescan when they overflow
        the slots) == skyrx_topk_threshold + skyrx_mask_gt, threshold bits too."""
        import torch
        from paper_2602_13509_b200 import rx

        v = (rng.standard_normal(n) ** 2 * 70).astype(np.float32)
        v[rng.integers(0, n, n // 50)] = np.float32(91.25)   # a tie-heavy threshold bin
        vt = torch.from_numpy(v).cuda()
        k = rx.topk_count(n)
        mask, thr = rx.topk_mask_device(vt, k, cap)
        thr0 = rx.topk_threshold_device(vt, k)
        assert bits(thr.cpu().numpy()) == bits(thr0.cpu().numpy())
        assert np.array_equal(mask.cpu().numpy().astype(bool), O.topk_mask(v, k))


# ----------------------------------------------------------------------------- the fused path
def check_detection(det, raw, t, gains=None):
    gains = np.ones(raw.shape[0]) if gains is None else gains
    want_stats, want_scores, want_mask = O.detect(raw, t.dark, t.coeff, gains)
    st = det.stats
    assert normwise(st.mu, want_stats.mu) < STATS_RTOL_FAST
    assert normwise(st.sigma, want_stats.sigma) < STATS_RTOL_FAST
    inv = normwise(st.sigma_inv, want_stats.sigma_inv)
    print(f"PARITY sigma_inv {inv:.3e} sigma {normwise(st.sigma, want_stats.sigma):.3e}")
    assert inv < INV_RTOL_FAST, inv
    assert st.ridge_used == want_stats.ridge_used
    rel = np.abs(det.scores - want_scores) / np.maximum(want_scores, 1e-12)
    assert rel.max() < SCORE_RTOL_FAST, rel.max()
    thr = O.topk_threshold(want_scores)
    differ = det.mask != want_mask
    near = np.abs(want_scores - thr) <= MASK_BAND * abs(thr)
    assert not (differ & ~near).any()
    return rel.max(), differ.sum()


class TestDetect:
    @pytest.mark.parametrize("seed,L,S,B,K", [(21, 48, 64, 70, 5), (23, 30, 40, 128, 5),
                                              (3, 40, 1024, 270, 8), (9, 17, 33, 5, 3)])
    def test_small_cubes_vs_oracle(self, P, seed, L, S, B, K):
        t = osynth.make_tables(seed, S, B, K)
        raw = osynth.generate_lines(t, 0, L)
        det = P.detect(raw_cube(P, raw), P.CalibrationTables(t.dark, t.coeff))
        check_detection(det, raw, t)

    def test_line_gains(self, P):
        t = osynth.make_tables(31, 64, 70)
        raw = osynth.generate_lines(t, 0, 50)
        gains = np.linspace(1.0, 8.0, 50)
        det = P.detect(raw_cube(P, raw, gains), P.CalibrationTables(t.dark, t.coeff))
        check_detection(det, raw, t, gains)

    @pytest.mark.parametrize("S,B", [(900, 70), (64, 70), (96, 48), (40, 16), (100, 80)])
    def test_tensor_core_score_matches_oracle_and_ffma(self, P, S, B):
        import torch

        from paper_2602_13509_b200 import _lib

        t = osynth.make_tables(41, S, B, 5)
        L = 70
        raw = osynth.generate_lines(t, 0, L)
        lib = _lib.load()
        rv = torch.from_numpy(raw).cuda()
        assert lib.skyrx_score_tc_supported(L, S, B, rv.data_ptr()) == 1
        tab = P.CalibrationTables(t.dark, t.coeff)
        plan_tc = P.DetectPlan(L, S, B)
        assert plan_tc.tc
        det_tc = P.detect(raw_cube(P, raw), tab, plan=plan_tc)
        plan_ff = P.DetectPlan(L, S, B)
        plan_ff.tc = False
        det_ff = P.detect(raw_cube(P, raw), tab, plan=plan_ff)
        check_detection(det_tc, raw, t)
        rel = np.abs(det_tc.scores - det_ff.scores) / np.maximum(det_ff.scores, 1e-12)
        assert rel.max() < 2e-5, rel.max()

    @pytest.mark.parametrize("S,B,L", [(900, 70, 300), (256, 128, 1100), (64, 96, 4200),
                                       (48, 16, 5600)])
    def test_exact_digit_score_kernel(self, P, monkeypatch, S, B, L):
        """score_tcs (integer deviations in two f16-exact digits, per-sample V_s)
        against the oracle; forced on for every B (by default it serves B > 80)."""
        from paper_2602_13509_b200 import _lib

        monkeypatch.setenv("SKYRX_B200_TCS", "1")
        t = osynth.make_tables(47, S, B, 5)
        raw = osynth.generate_lines(t, 0, L)
        plan = P.DetectPlan(L, S, B)
        assert plan.tcs
        assert L * S >= P.rx.TC_MIN_PIXELS
        det = P.detect(raw_cube(P, raw), P.CalibrationTables(t.dark, t.coeff), plan=plan)
        assert plan.used_raw[0]
        assert int(plan.ds.flags[0].item()) & 16 == 0
        check_detection(det, raw, t)

    @pytest.mark.parametrize("S,B,L", [(1024, 270, 70), (128, 160, 300), (64, 144, 129)])
    def test_wide_exact_digit_score_kernel(self, P, S, B, L):
        """score_tcw (128 < B <= 272: V_s streamed in N-blocks) against the oracle."""
        t = osynth.make_tables(49, S, B, 8)
        raw = osynth.generate_lines(t, 0, L)
        plan = P.DetectPlan(L, S, B)
        assert plan.tcw
        det = P.detect(raw_cube(P, raw), P.CalibrationTables(t.dark, t.coeff), plan=plan)
        fl = int(plan.ds.flags[0].item())
        assert (fl & 12) == 8 or (fl & 192) == 128  # no-clamp proof from the moments pass
        assert not fl & (16 | 32)                   # the exact-digit kernel applied
        check_detection(det, raw, t)

    def test_wide_kernel_without_clamp_proof_rescores(self, P):
        S, B, L = 128, 160, 100
        t = osynth.make_tables(50, S, B, 8)
        raw = osynth.generate_lines(t, 0, L).copy()
        raw[3, 4, 5] = 0  # below dark: clamps
        plan = P.DetectPlan(L, S, B)
        det = P.detect(raw_cube(P, raw), P.CalibrationTables(t.dark, t.coeff), plan=plan)
        fl = int(plan.ds.flags[0].item())
        assert fl & (4 | 64)  # the clamp was seen by whichever moments pass ran
        check_detection(det, raw, t)

    def test_exact_digit_kernel_rejects_wide_counts(self, P, monkeypatch):
        """Counts >= 4096 (not 12-bit) flag the digit kernel; detect() rescores with
        the general tensor-core kernel and still matches the oracle."""
        monkeypatch.setenv("SKYRX_B200_TCS", "1")
        S, B, L = 900, 70, 300
        t = osynth.make_tables(48, S, B, 5)
        raw = osynth.generate_lines(t, 0, L).copy()
        raw[7, 100:140, 3] = 5000
        raw[201, 5, :] = 4600
        plan = P.DetectPlan(L, S, B)
        det = P.detect(raw_cube(P, raw), P.CalibrationTables(t.dark, t.coeff), plan=plan)
        assert int(plan.ds.flags[0].item()) & 16
        check_detection(det, raw, t)

    def test_detect_batch_matches_detect(self, P):
        """The pipelined host-buffer batch (two device slots, copy stream) returns what
        detect() returns cube by cube, including a cube that needs the general path."""
        S, B, L = 900, 70, 64
        tabs, raws = [], []
        for i in range(5):
            t = osynth.make_tables(60 + i, S, B, 5)
            raw = osynth.generate_lines(t, 0, L).copy()
            if i == 3:
                raw[5, 6, 7] = 0  # clamps: redone through detect()
            tabs.append(P.CalibrationTables(t.dark, t.coeff))
            raws.append(raw_cube(P, raw))
        got = P.detect_batch(raws, tabs)
        for g, r, tb in zip(got, raws, tabs):
            want = P.detect(r, tb)
            assert np.array_equal(g.scores, want.scores)
            assert np.array_equal(g.mask, want.mask)
            assert g.threshold == want.threshold and g.max_score == want.max_score
            assert np.array_equal(g.stats.sigma_inv, want.stats.sigma_inv)

    @pytest.mark.parametrize("L", [1, 33, 129])
    def test_tensor_core_score_schedule_edges(self, P, L):
        """Fewer tiles than sample blocks, and ragged narrow-block tiles (2-D TMA box
        past the last line) against the FFMA kernel."""
        S, B = 900, 70
        t = osynth.make_tables(43, S, B, 5)
        raw = osynth.generate_lines(t, 0, L)
        tab = P.CalibrationTables(t.dark, t.coeff)
        det_tc = P.detect(raw_cube(P, raw), tab, plan=P.DetectPlan(L, S, B))
        plan_ff = P.DetectPlan(L, S, B)
        plan_ff.tc = False
        det_ff = P.detect(raw_cube(P, raw), tab, plan=plan_ff)
        rel = np.abs(det_tc.scores - det_ff.scores) / np.maximum(det_ff.scores, 1e-12)
        assert rel.max() < 2e-5, rel.max()

    @pytest.mark.parametrize("S,B,L,gain", [(900, 70, 300, 1.0), (64, 70, 4100, 2.5),
                                            (96, 48, 2800, 1.0), (40, 16, 6600, 1.0),
                                            (1024, 128, 260, 1.0), (128, 79, 2100, 0.75),
                                            (1024, 270, 300, 1.0), (128, 160, 2100, 0.75),
                                            (64, 150, 4100, 1.0), (900, 70, 2100, 1.0)])
    def test_raw_byte_moments(self, P, S, B, L, gain):
        """Constant line gain: exact integer byte Grams on the tensor cores."""
        from paper_2602_13509_b200 import _lib
        from paper_2602_13509_b200.rx import TC_MIN_PIXELS
        from paper_2602_13509_b200.synth import Scene

        assert L * S >= TC_MIN_PIXELS
        rv = Scene(43, S, B, 5).generate(0, L)
        raw = rv.cpu().numpy()
        t = osynth.make_tables(43, S, B, 5)
        assert _lib.load().skyrx_stats_raw_supported(L, S, B, rv.data_ptr()) == 1
        gains = np.full(L, gain)
        det = P.detect(raw_cube(P, raw, gains), P.CalibrationTables(t.dark, t.coeff))
        check_detection(det, raw, t, gains)
        ref = O.compute_stats(O.apply_calibration(raw, t.dark, t.coeff, gains))
        # exact integer Gram of the exact radiance (r - d) c / g.  The reference sums
        # f32-ROUNDED radiance: fl(r - d) carries an offset fixed per (sample, band,
        # binade of r - d), which correlates with x and moves sigma by ~1e-8
        # relative; that reference-side rounding is the whole residual here.
        assert normwise(det.stats.sigma, ref.sigma) < 1e-7
        assert normwise(det.stats.mu, ref.mu) < 1e-8

    @pytest.mark.parametrize("S,B,L", [(900, 70, 300), (96, 48, 2800), (128, 79, 2100)])
    def test_quantised_moments_varying_gains(self, P, S, B, L):
        """Varying line gains: dithered int8-digit Gram on the tensor cores."""
        from paper_2602_13509_b200.synth import Scene

        raw = Scene(44, S, B, 5).generate(0, L).cpu().numpy()
        t = osynth.make_tables(44, S, B, 5)
        gains = 1.0 + 0.5 * np.sin(np.arange(L) / 17.0) ** 2
        plan = P.DetectPlan(L, S, B)
        assert plan.tc_stats
        det = P.detect(raw_cube(P, raw, gains), P.CalibrationTables(t.dark, t.coeff), plan=plan)
        check_detection(det, raw, t, gains)
        ref = O.compute_stats(O.apply_calibration(raw, t.dark, t.coeff, gains))
        # quantiser noise only (dithered, unbiased): far below the 1e-5 contract
        assert normwise(det.stats.sigma, ref.sigma) < 1e-6
        assert normwise(det.stats.mu, ref.mu) < 1e-7

    def test_quantiser_range_fallback(self, P, rng):
        # varying gains + a flat cube with one far outlier outside the shift sample
        # overflow the int8 quantiser; detect() must notice and redo the fit in f64
        L, S, B = 300, 900, 70
        raw = (1000 + rng.integers(-3, 4, (L, S, B))).astype(np.uint16)
        assert (1 * S + 100) % ((L * S) // 4096) != 0   # not a sampled pixel
        raw[1, 100] = 4000
        dark = np.full((S, B), 100.0, np.float32)
        coeff = np.ones((S, B), np.float32)
        gains = np.ones(L)
        gains[7] = 2.0
        det = P.detect(raw_cube(P, raw, gains), P.CalibrationTables(dark, coeff))
        rad = O.apply_calibration(raw, dark, coeff, gains)
        ref = O.compute_stats(rad)
        assert normwise(det.stats.sigma, ref.sigma) < 1e-12
        assert normwise(det.stats.mu, ref.mu) < 1e-12
        want = O.rx_scores(rad, ref)
        assert (np.abs(det.scores - want) / np.maximum(want, 1e-12)).max() < 1e-4
        assert det.mask[1, 100]

    @pytest.mark.parametrize("S,B,L", [(900, 70, 2100), (64, 150, 4100), (128, 79, 700)])
    def test_own_shift_equals_given_shift(self, P, S, B, L):
        """skyrx_stats_raw_own_shift centres on f32(mean) itself; the same call with that
        shift passed in (skyrx_stats_raw) gives the same moments, and the shift is the
        f32 of the oracle's mean."""
        import torch
        from paper_2602_13509_b200 import _lib, _dev
        from paper_2602_13509_b200.synth import Scene

        sc = Scene(47, S, B, 5)
        rv = sc.generate(0, L)
        d, c = torch.from_numpy(sc.dark).cuda(), torch.from_numpy(sc.coeff).cuda()
        f64 = torch.float64
        ws_bytes = int(_lib.load().skyrx_stats_raw_workspace(B))
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
        shift = torch.zeros(B, dtype=f64, device="cuda")
        m1 = torch.zeros(1 + B + B * B, dtype=f64, device="cuda")
        m2 = torch.zeros_like(m1)
        fl = torch.zeros(1, dtype=torch.int32, device="cuda")
        args = (rv.data_ptr(), L, S, B, d.data_ptr(), c.data_ptr(), 1.0)
        _lib.call("skyrx_stats_raw_own_shift", *args, shift.data_ptr(), m1.data_ptr(),
                  fl.data_ptr(), ws.data_ptr(), ws_bytes, _dev.stream_ptr())
        _lib.call("skyrx_stats_raw", *args, shift.data_ptr(), m2.data_ptr(), fl.data_ptr(),
                  ws.data_ptr(), ws_bytes, _dev.stream_ptr())
        torch.cuda.synchronize()
        assert torch.equal(m1, m2)
        raw = rv.cpu().numpy()
        ref = O.compute_stats(O.apply_calibration(raw, sc.dark, sc.coeff, np.ones(L)))
        assert np.array_equal(shift.cpu().numpy(), ref.mu.astype(np.float32).astype(np.float64)) \
            or normwise(shift.cpu().numpy(), ref.mu) < 1e-7
        n = m1[0].item()
        mu = shift.cpu().numpy() + m1[1:1 + B].cpu().numpy() / n
        assert normwise(mu, ref.mu) < 1e-8

    def test_raw_path_clamp_corrected(self, P):
        # a value below its dark level clamps to 0 (calibrate.py:99): the raw-byte
        # algebra no longer holds for that pixel, so the clamped pixels' exact
        # corrections are added in the same call (clamp_fix_kernel; flags 4 | 256)
        # instead of redoing the cube in f64
        L, S, B = 300, 900, 70
        t = osynth.make_tables(45, S, B, 5)
        raw = osynth.generate_lines(t, 0, L)
        raw[5, 17, 3] = 20      # dark ~ 100 -> clamps
        plan = P.DetectPlan(L, S, B)
        det = P.detect(raw_cube(P, raw), P.CalibrationTables(t.dark, t.coeff), plan=plan)
        assert int(plan.ds.flags[0].item()) & (4 | 256) == (4 | 256)
        assert plan.used_raw[0]
        rad = O.apply_calibration(raw, t.dark, t.coeff, np.ones(L))
        assert rad[5, 17, 3] == 0.0
        ref = O.compute_stats(rad)
        exact = O.compute_stats_exact(raw, t.dark, t.coeff, np.ones(L))
        assert normwise(det.stats.sigma, exact.sigma) < 1e-12   # exact correction
        assert normwise(det.stats.sigma, ref.sigma) < 1e-7
        check_detection(det, raw, t)

    @pytest.mark.parametrize("S,B,L", [(900, 70, 2100), (512, 128, 1100), (64, 40, 9000)])
    def test_sparse_and_dead_pixel_clamps(self, P, S, B, L):
        """0.01 % random sub-dark counts plus one dead detector element (a whole
        (sample, band) column below dark): corrected moments, then scores (score_tc
        clamps natively; B > 80 rescores through the general kernel)."""
        rng = np.random.default_rng(S + B)
        t = osynth.make_tables(46, S, B, 5)
        raw = osynth.generate_lines(t, 0, L).copy()
        n = raw.size
        idx = rng.choice(n, max(1, n // 10000), replace=False)
        raw.reshape(-1)[idx] = rng.integers(0, 60, idx.size)
        raw[:, S // 3, B // 2] = 5
        plan = P.DetectPlan(L, S, B)
        det = P.detect(raw_cube(P, raw), P.CalibrationTables(t.dark, t.coeff), plan=plan)
        assert int(plan.ds.flags[0].item()) & (4 | 256) == (4 | 256)
        exact = O.compute_stats_exact(raw, t.dark, t.coeff, np.ones(L))
        assert normwise(det.stats.sigma, exact.sigma) < 1e-11
        assert normwise(det.stats.mu, exact.mu) < 1e-12
        check_detection(det, raw, t)

    @pytest.mark.parametrize("S,B,L", [(64, 70, 700), (40, 33, 333), (64, 96, 700), (48, 80, 300),
                                       (32, 128, 520)])
    def test_clamp_marking_threshold_edges(self, P, S, B, L):
        """The scan warps mark a pixel iff some count r has (float)r < dark, tested as
        r < ceil(dark) on u16 pairs: integer and fractional darks at r = dark - 1, dark,
        dark + 1, a dark <= 0 (never clamps) and a dark > 65535 (every count clamps),
        in full and partial tiles, in box 0 and past byte 128.  calibrate.py:99."""
        t = osynth.make_tables(48, S, B, 5)
        dark = t.dark.copy()
        raw = osynth.generate_lines(t, 0, L).copy()
        dark[3, 2] = 100.0       # integer dark: 99 clamps, 100 and 101 do not
        dark[5, B - 1] = 100.5   # fractional (the last band: past byte 128 when B > 64)
        dark[7, 0] = 0.0
        dark[8, 1] = -5.0
        dark[9, B // 2] = 70000.0  # above every u16 count: the whole column clamps
        raw[0:3, 3, 2] = (99, 100, 101)
        raw[130:133, 5, B - 1] = (100, 101, 102)
        raw[L - 1, 5, B - 1] = 7       # in the partial last tile
        raw[200, 7, 0] = 0
        raw[201, 8, 1] = 0
        plan = P.DetectPlan(L, S, B)
        det = P.detect(raw_cube(P, raw), P.CalibrationTables(dark, t.coeff), plan=plan)
        assert int(plan.ds.flags[0].item()) & (4 | 256) == (4 | 256)
        exact = O.compute_stats_exact(raw, dark, t.coeff, np.ones(L))
        assert normwise(det.stats.sigma, exact.sigma) < 1e-11
        assert normwise(det.stats.mu, exact.mu) < 1e-12
        rad = O.apply_calibration(raw, dark, t.coeff, np.ones(L))
        assert rad[0, 3, 2] == 0.0 and rad[1, 3, 2] == 0.0 and rad[2, 3, 2] > 0.0
        assert rad[130, 5, B - 1] == 0.0 and rad[131, 5, B - 1] > 0.0
        assert (rad[:, 9, B // 2] == 0.0).all()

    @pytest.mark.parametrize("S,B,L", [(900, 70, 2100), (128, 128, 1100)])
    def test_dead_element_only(self, P, S, B, L):
        """One dead detector element (a whole (sample, band) column below dark) and nothing
        else: few units clamp, so the marking reads only the flagged units (the per-unit
        marking); the corrected moments are exact."""
        t = osynth.make_tables(47, S, B, 5)
        raw = osynth.generate_lines(t, 0, L).copy()
        raw[:, S // 2, B // 3] = 3
        raw[L // 2, 5, 1] = 0  # and one isolated sub-dark count elsewhere
        plan = P.DetectPlan(L, S, B)
        det = P.detect(raw_cube(P, raw), P.CalibrationTables(t.dark, t.coeff), plan=plan)
        assert int(plan.ds.flags[0].item()) & (4 | 256) == (4 | 256)
        exact = O.compute_stats_exact(raw, t.dark, t.coeff, np.ones(L))
        assert normwise(det.stats.sigma, exact.sigma) < 1e-11
        assert normwise(det.stats.mu, exact.mu) < 1e-12
        check_detection(det, raw, t)

    def test_deterministic(self, P):
        t = osynth.make_tables(1, 900, 70)
        raw = osynth.generate_lines(t, 0, 128)
        cube = raw_cube(P, raw)
        tab = P.CalibrationTables(t.dark, t.coeff)
        a, b = P.detect(cube, tab), P.detect(cube, tab)
        assert np.array_equal(bits(a.scores), bits(b.scores))
        assert np.array_equal(a.stats.sigma, b.stats.sigma)
        assert np.array_equal(a.mask, b.mask)

    @pytest.mark.slow
    def test_c1_full_size_vs_oracle(self, P):
        c = osynth.CONFIGS["c1"]
        t = osynth.make_tables(c["seed"], c["samples"], c["bands"], c["components"])
        from paper_2602_13509_b200.synth import Scene

        raw = Scene(c["seed"], c["samples"], c["bands"], c["components"]).generate(
            0, c["lines"]).cpu().numpy()
        det = P.detect(raw_cube(P, raw), P.CalibrationTables(t.dark, t.coeff))
        worst, ndiff = check_detection(det, raw, t)
        assert det.mask.sum() <= osynth.CONFIGS["c1"]["lines"] * 900 // 1000 + 1
