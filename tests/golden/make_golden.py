"""Regenerate tests/golden/*.npz by running the REAL reference package.

    NUMBA_CACHE_DIR=/tmp/numba PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py [/root/reference/pkg/src]

Only runs in the build container (the reference tree is not shipped to GPU
boxes); the committed .npz files are what tests read.  Every fixture is the
output of the reference's own functions (skyrx.calibrate / skyrx.rx /
skyrx._accel) on seeded inputs, so tests/test_oracle.py pins the oracle to
the reference and the -m gpu tests pin the CUDA path to the same numbers.
"""

from __future__ import annotations

import hashlib
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
REF_SRC = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF_SRC)
sys.path.insert(0, str(ROOT))

from skyrx import _accel  # noqa: E402
from skyrx.calibrate import CalibrationTables, apply_calibration, calibrate_bin_rgb  # noqa: E402
from skyrx.cube import InsSample, LineMeta, RadianceCube, RawCube, ScoreMap  # noqa: E402
from skyrx.rx import compute_stats, normalize_scores, rx_scores, threshold_scores  # noqa: E402
from skyrx.scene import band_grid  # noqa: E402

from oracle import synth  # noqa: E402  (generator only; outputs below come from skyrx)


AIR_BANDS, AIR_LINES, AIR_CUBES, AIR_SEED = 44, 50, 3, 2602


def air_inputs(tables_cls, raw_cls, band_grid_fn, metas_fn):
    """The run_air fixture's inputs (shared with tests/test_gpu_air.py): AIR_CUBES cubes of
    AIR_LINES x 900 x AIR_BANDS from one synthetic scene, per-line gains varying."""
    st = synth.make_tables(AIR_SEED, 900, AIR_BANDS)
    wl = band_grid_fn(AIR_BANDS)
    cubes = []
    for c in range(AIR_CUBES):
        raw = synth.generate_lines(st, c * AIR_LINES, AIR_LINES)
        gains = [1.0 + 0.25 * ((c + i) % 3) for i in range(AIR_LINES)]
        cubes.append(raw_cls(raw, wl, metas_fn(gains)))
    return {"cubes": cubes, "tables": tables_cls(st.dark, st.coeff)}


def metas(gains):
    out = []
    for i, g in enumerate(gains):
        t = 1_600_000_000_000_000 + i * 4016
        ins = InsSample(t - 1000, 35.0, -90.0, 40.0, 0.0, 0.0, 0.0)
        ins2 = InsSample(t + 4000, 35.0, -90.0, 40.0, 0.0, 0.0, 0.0)
        out.append(LineMeta(t, float(g), ins, ins2))
    return tuple(out)


def rad(values, gain=2.0):
    values = np.asarray(values, np.float32)
    return RadianceCube(values, np.linspace(400.0, 1000.0, values.shape[2]),
                        metas([gain] * values.shape[0]))


def stats_case(prefix, cube, store, extra_threshold=None):
    st = compute_stats(cube)
    sc = rx_scores(cube, st)
    store[f"{prefix}/values"] = cube.values
    store[f"{prefix}/mu"] = st.mu
    store[f"{prefix}/sigma"] = st.sigma
    store[f"{prefix}/sigma_inv"] = st.sigma_inv
    store[f"{prefix}/chol"] = st.chol_lower
    store[f"{prefix}/ridge"] = np.float64(st.ridge_used)
    store[f"{prefix}/scores"] = sc.values
    norm = normalize_scores(sc)
    store[f"{prefix}/norm"] = norm.values
    if extra_threshold is not None:
        store[f"{prefix}/mask_t"] = threshold_scores(norm, extra_threshold)


def main():
    rng = np.random.default_rng(20240901)

    # ---------------------------------------------------------------- calibration
    cal = {}
    raw = rng.integers(0, 4096, (6, 7, 24), dtype=np.uint16)
    dark = rng.uniform(0, 120, (7, 24)).astype(np.float32)
    coeff = rng.uniform(0.5, 2.0, (7, 24)).astype(np.float32)
    gains = rng.uniform(1.0, 8.0, 6).astype(np.float32).astype(np.float64)
    out = apply_calibration(RawCube(raw, np.linspace(400, 1000, 24), metas(gains)),
                            CalibrationTables(dark, coeff))
    cal.update({"rand/raw": raw, "rand/dark": dark, "rand/coeff": coeff,
                "rand/gains": gains, "rand/out": out.values})

    raw = np.full((1, 1, 24), 100, np.uint16)
    out = apply_calibration(RawCube(raw, np.linspace(400, 1000, 24), metas([4.0])),
                            CalibrationTables(np.full((1, 24), 10.0, np.float32),
                                              np.full((1, 24), 2.0, np.float32)))
    cal["bydef/out"] = out.values  # 45.0 everywhere (test_calibrate.py:42-48)

    t = synth.make_tables(11, 96, 70)
    raw = synth.generate_lines(t, 0, 32)
    g = np.ones(32)
    g[5] = 3.0
    g[17] = 0.37
    out = apply_calibration(RawCube(raw, np.linspace(400, 1000, 70), metas(g)),
                            CalibrationTables(t.dark, t.coeff))
    cal.update({"synth/raw": raw, "synth/gains": g, "synth/out": out.values})

    # fused calibrate -> discard -> bin -> rgb
    for name, (shape, wl, factor) in {
        "b300": ((4, 5, 300), band_grid(300), 4),
        "b44": ((5, 6, 44), band_grid(44), 4),
        "b340f8": ((3, 4, 340), band_grid(340), 8),
    }.items():
        raw = rng.integers(0, 4096, shape, dtype=np.uint16)
        dark = rng.uniform(0, 40, shape[1:]).astype(np.float32)
        coeff = rng.uniform(0.5, 1.5, shape[1:]).astype(np.float32)
        gains = rng.uniform(1.0, 4.0, shape[0]).astype(np.float32).astype(np.float64)
        cube, rgb = calibrate_bin_rgb(RawCube(raw, wl, metas(gains)),
                                      CalibrationTables(dark, coeff), factor=factor,
                                      chunk_lines=2)
        cal.update({f"{name}/raw": raw, f"{name}/wl": np.asarray(wl), f"{name}/dark": dark,
                    f"{name}/coeff": coeff, f"{name}/gains": gains, f"{name}/factor": factor,
                    f"{name}/out": cube.values, f"{name}/centers": cube.wavelengths_nm,
                    f"{name}/rgb": rgb})
    np.savez_compressed(HERE / "calibrate.npz", **cal)

    # ---------------------------------------------------------------- statistics + scores
    st = {}
    vals = (np.arange(48, dtype=np.float32).reshape(4, 4, 3) * 7 % 23).astype(np.float32)
    stats_case("hand", rad(vals), st)
    stats_case("mean0", rad(np.array([1, 3, 2, 2], np.float32).reshape(2, 2, 1)), st)
    stats_case("hand1", rad(np.array([0, 0, 0, 4], np.float32).reshape(2, 2, 1)), st)
    stats_case("ident", rad(np.full((4, 4, 3), 9.0)), st)
    base = np.arange(16, dtype=np.float32)
    stats_case("rank1", rad(np.stack([base, 2 * base], axis=1).reshape(4, 4, 2)), st)
    stats_case("normal", rad(rng.normal(80, 6, (12, 11, 6)).astype(np.float32)), st)
    stats_case("chi2", rad(rng.normal(0, 1, (100, 4, 4)).astype(np.float32)), st)
    r7 = np.random.default_rng(7)           # test_acceptance.py:28-42 style cubes
    for trial in range(6):
        lines, samples, bands = int(r7.integers(8, 33)), int(r7.integers(8, 33)), int(r7.integers(2, 9))
        b = r7.normal(r7.uniform(20, 200), r7.uniform(2, 15), (lines, samples, bands))
        stats_case(f"acc{trial}", rad(np.abs(b).astype(np.float32)), st)
    t = synth.make_tables(21, 64, 70)
    raw = synth.generate_lines(t, 0, 48)
    cube = apply_calibration(RawCube(raw, np.linspace(400, 1000, 70), metas([1.0] * 48)),
                             CalibrationTables(t.dark, t.coeff))
    st["synth70/raw"] = raw
    stats_case("synth70", cube, st, extra_threshold=0.11)
    t = synth.make_tables(23, 40, 128)
    raw = synth.generate_lines(t, 100, 30)
    cube = apply_calibration(RawCube(raw, np.linspace(400, 1000, 128), metas([1.0] * 30)),
                             CalibrationTables(t.dark, t.coeff))
    st["synth128/raw"] = raw
    stats_case("synth128", cube, st, extra_threshold=0.11)
    np.savez_compressed(HERE / "stats.npz", **st)

    # ---------------------------------------------------------------- kernel slot
    acc = {}
    n, b = 4000, 12
    px = rng.normal(50, 4, (n, b)).astype(np.float32)
    cov = np.cov(px.astype(np.float64).T) + np.eye(b) * 1e-6
    mu = px.mean(axis=0, dtype=np.float64)
    chol = np.linalg.cholesky(cov)
    acc.update({"px": px, "mu": mu, "chol": chol,
                "numba": _accel.mahalanobis_sq(px, mu, chol),
                "numpy": _accel.mahalanobis_sq_numpy(px, mu, chol, chunk=997),
                "has_numba": np.bool_(_accel.HAS_NUMBA)})
    np.savez_compressed(HERE / "accel.npz", **acc)

    # ---------------------------------------------------------------- normalize / threshold
    nt = {}
    sm = ScoreMap(rng.random((6, 6)) * 5)
    nt["rand/values"] = sm.values
    nt["rand/norm"] = normalize_scores(sm).values
    nt["rand/mask037"] = threshold_scores(normalize_scores(sm), 0.37)
    v = np.array([[0.5, 8.0], [1.0, 0.0]], np.float32)
    nt["small/values"] = v
    nt["small/norm"] = normalize_scores(ScoreMap(v)).values
    nt["small/mask1"] = threshold_scores(normalize_scores(ScoreMap(v)), 1.0)
    nt["small/mask0"] = threshold_scores(normalize_scores(ScoreMap(v)), 0.0)
    # f32 rounding of t (NEP 50): t sits just below v in f64 but rounds up to v in f32,
    # so the reference's compare `v > t` is False (it would be True in f64)
    v = np.nextafter(np.float32(0.11), np.float32(1))
    edge = np.array([[v, np.float32(0.11), 1.0]], np.float32)
    t_edge = float(v) - 1e-12
    nt["edge/values"] = edge
    nt["edge/t"] = np.float64(t_edge)
    nt["edge/mask"] = threshold_scores(ScoreMap(edge), t_edge)
    np.savez_compressed(HERE / "normalize.npz", **nt)

    # ---------------------------------------------------------------- link payload
    from skyrx.datalink import encode_scores_half, pack_rgb565, packetize_cube
    lk = {}
    rgb = rng.random((900, 3)).astype(np.float32) * np.float32(40.0)
    sc = (rng.random(900) ** 3 * 500).astype(np.float32)
    # round-half-up edges: exact multiples of max/levels and their half steps
    rgb[:6, 0] = np.float32(40.0) * np.array([0, 1, 0.5 / 31, 1.5 / 31, 30.5 / 31, 2.0 / 31],
                                              np.float32)
    sc[:4] = np.array([0.0, 500.0, 1e-30, 499.99997], np.float32)
    lk["row/rgb"], lk["row/scores"] = rgb, sc
    lk["row/rgb565"] = pack_rgb565(rgb, 40.0, 37.5, 12.25)
    lk["row/half"] = encode_scores_half(sc, 500.0)
    lk["row/half_zero_max"] = encode_scores_half(sc, 0.0)
    lk["row/rgb565_zero_max"] = pack_rgb565(rgb, 0.0, 37.5, -1.0)
    lines = 3
    cube_rgb = (rng.random((lines, 900, 3)) * 30).astype(np.float32)
    cube_sc = (rng.random((lines, 900)) ** 4 * 900).astype(np.float32)
    pk = packetize_cube(7, cube_rgb, cube_sc, metas([1.0] * lines))
    lk["cube/rgb"], lk["cube/scores"] = cube_rgb, cube_sc
    lk["cube/packets"] = np.frombuffer(b"".join(pk), np.uint8)
    np.savez_compressed(HERE / "datalink.npz", **lk)

    # ---------------------------------------------------------------- GF(256) erasure code
    from skyrx import fec
    from skyrx.datalink import frames_for_cube

    fc = {"gf_log": fec.GF_LOG, "gf_exp": fec.GF_EXP}
    code = fec.ErasureCode(50, 25)
    fc["matrix_50_25"] = code.matrix
    fc["matrix_4_3"] = fec.ErasureCode(4, 3).matrix
    fc["matrix_1_0"] = fec.ErasureCode(1, 0).matrix
    fc["matrix_200_56"] = fec.ErasureCode(200, 56).matrix
    r2 = np.random.default_rng(2024)
    mat = r2.integers(0, 256, (7, 13), dtype=np.uint8)
    mat[0, :] = 0
    mat[:, 3] = 0
    data = r2.integers(0, 256, (13, 333), dtype=np.uint8)
    data[5, :] = 0
    data[:, 17] = 0
    fc["mm/mat"], fc["mm/data"] = mat, data
    fc["mm/out"] = _accel.gf256_matmul_numpy(mat, data, fec.GF_LOG, fec.GF_EXP)
    m6 = np.random.default_rng(3).integers(0, 256, (6, 6), dtype=np.uint8)
    m6 += np.eye(6, dtype=np.uint8)
    fc["inv/m"], fc["inv/minv"] = m6, fec.gf_mat_inv(m6)
    payloads = [r2.integers(0, 256, 211, dtype=np.uint8).tobytes() for _ in range(50)]
    coded = payloads + code.encode(payloads)
    fc["enc/coded"] = np.frombuffer(b"".join(coded), np.uint8).reshape(75, 211)
    keeps = [np.arange(25, 75)] + [np.sort(r2.permutation(75)[:50]) for _ in range(6)]
    keeps += [np.sort(r2.permutation(75)[:49]), np.arange(0, 50), np.sort(r2.permutation(75)[:60])]
    for c, keep in enumerate(keeps):
        rec, rep = code.decode([(int(i), coded[int(i)]) for i in keep])
        fc[f"dec{c}/keep"] = keep.astype(np.int64)
        fc[f"dec{c}/slots"] = np.array(sorted(rec), np.int64)
        fc[f"dec{c}/data"] = np.frombuffer(b"".join(rec[i] for i in sorted(rec)), np.uint8)
        fc[f"dec{c}/report"] = np.array([len(rep.received), len(rep.recovered), len(rep.missing)])
        fc[f"dec{c}/recovered"] = np.array(rep.recovered, np.int64)
        fc[f"dec{c}/missing"] = np.array(rep.missing, np.int64)
    pk = [r2.integers(0, 256, 97, dtype=np.uint8).tobytes() for _ in range(100)]
    frames = frames_for_cube(3, pk)
    fc["frames/packets"] = np.frombuffer(b"".join(pk), np.uint8)
    fc["frames/frames"] = np.frombuffer(b"".join(frames), np.uint8)
    fc["frames/lengths"] = np.array([len(f) for f in frames], np.int64)
    np.savez_compressed(HERE / "fec.npz", **fc)

    # ---------------------------------------------------------------- air pipeline (run_air)
    # cubes from oracle/synth (tests regenerate them bit-identically), run through the
    # reference's own four-stage pipeline; what is stored is the reference's output.
    from skyrx.formats import write_cube
    from skyrx.pipeline import FlightData, PipelineConfig, run_air

    ap = air_inputs(CalibrationTables, RawCube, band_grid, metas)
    config = PipelineConfig(bands=AIR_BANDS, samples=900, bin_factor=4, queue_depth=2)
    res = run_air(config, FlightData(cubes=ap["cubes"], track=None, masks=[],
                                     tables=ap["tables"]))
    assert not res.dropped, res.dropped
    ag = {"frames": np.frombuffer(b"".join(res.frames), np.uint8),
          "lengths": np.array([len(f) for f in res.frames], np.int64)}
    for c, (sc, rgb) in enumerate(zip(res.scores, res.rgb)):
        ag[f"scores{c}"] = sc.values
        ag[f"rgb{c}_sha256"] = np.frombuffer(
            hashlib.sha256(np.ascontiguousarray(rgb, np.float32).tobytes()).digest(), np.uint8)
    tiny = RawCube(np.arange(3 * 4 * 5, dtype=np.uint16).reshape(3, 4, 5) * 7,
                   band_grid(25)[:5], metas([1.0, 0.5, 2.0]))
    import tempfile

    with tempfile.TemporaryDirectory() as td:
        write_cube(Path(td) / "t.hsc", tiny)
        ag["tiny_hsc"] = np.frombuffer((Path(td) / "t.hsc").read_bytes(), np.uint8)
    np.savez_compressed(HERE / "air.npz", **ag)
    print("wrote", sorted(p.name for p in HERE.glob("*.npz")))


if __name__ == "__main__":
    main()
