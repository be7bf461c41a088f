"""The air pipeline on CUDA streams against the reference's own run_air
output (tests/golden/air.npz, made by tests/golden/make_golden.py on the same synthetic
cubes), plus the reference's pipeline tests: queue-depth invariance, save stage, poisoned
cube isolation, and .hsc ingest."""

import dataclasses
import hashlib
import struct
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import skyrx_oracle as O
from oracle import synth

pytestmark = pytest.mark.gpu

AIR_BANDS, AIR_LINES, AIR_CUBES, AIR_SEED = 44, 50, 3, 2602   # = make_golden.py


def band_grid(bands):
    """scene.py:145-158 geometry: bands-20 centres across [400, 1000] nm, 10 beyond each end."""
    inner = np.linspace(400.0, 1000.0, bands - 20)
    step = inner[1] - inner[0]
    g = np.concatenate([400.0 - step * np.arange(10, 0, -1), inner,
                        1000.0 + step * np.arange(1, 11)])
    return g.astype(np.float32).astype(np.float64)


def metas(P, gains):
    out = []
    for i, g in enumerate(gains):
        t = 1_600_000_000_000_000 + i * 4016
        out.append(P.LineMeta(t, float(g), P.InsSample(t - 1000, 35.0, -90.0, 40.0, 0, 0, 0),
                              P.InsSample(t + 4000, 35.0, -90.0, 40.0, 0, 0, 0)))
    return tuple(out)


@pytest.fixture(scope="module")
def P():
    import paper_2602_13509_b200 as P
    from paper_2602_13509_b200 import build

    build.build()
    return P


@pytest.fixture(scope="module")
def flight(P):
    st = synth.make_tables(AIR_SEED, 900, AIR_BANDS)
    wl = band_grid(AIR_BANDS)
    cubes = []
    for c in range(AIR_CUBES):
        gains = [1.0 + 0.25 * ((c + i) % 3) for i in range(AIR_LINES)]
        cubes.append(P.RawCube(synth.generate_lines(st, c * AIR_LINES, AIR_LINES), wl,
                               metas(P, gains)))
    return SimpleNamespace(cubes=cubes, tables=P.CalibrationTables(st.dark, st.coeff))


def config(**kw):
    return SimpleNamespace(**{"bin_factor": 4, "queue_depth": 2, "out_dir": None, **kw})


@pytest.fixture(scope="module")
def result(P, flight):
    from paper_2602_13509_b200.air import run_air

    return run_air(config(), flight)


def _split(frames):
    return [struct.unpack_from("<IBBH", f) + (f[8:],) for f in frames]


def test_matches_reference_run_air(result, golden):
    g = golden["air"]
    assert result.dropped == []
    assert [len(f) for f in result.frames] == g["lengths"].tolist()
    ref, off = [], 0
    for n in g["lengths"]:
        ref.append(g["frames"][off:off + n].tobytes())
        off += n
    for c in range(AIR_CUBES):
        rgb = np.ascontiguousarray(result.rgb[c], np.float32).tobytes()
        assert hashlib.sha256(rgb).digest() == g[f"rgb{c}_sha256"].tobytes()   # bit-exact
        np.testing.assert_allclose(result.scores[c].values, g[f"scores{c}"], rtol=1e-6)
    mine, theirs = _split(result.frames), _split(ref)
    exact, ulp = 0, 0
    for (gid, idx, kind, _, pay), (rgid, ridx, rkind, _, rpay) in zip(mine, theirs):
        assert (gid, idx, kind) == (rgid, ridx, rkind)
        if kind == 1:
            continue
        a, b = np.frombuffer(pay, np.uint8), np.frombuffer(rpay, np.uint8)
        assert a[:128].tobytes() == b[:128].tobytes()            # headers incl. maxima
        wa, wb = a[128:].view("<u2").reshape(-1, 2), b[128:].view("<u2").reshape(-1, 2)
        assert np.array_equal(wa[:, 0], wb[:, 0])               # RGB565 bit-exact
        d = np.abs(wa[:, 1].astype(np.int32) - wb[:, 1].astype(np.int32))
        assert d.max() <= 1                                      # half(sqrt(s/max)): 1 ulp
        exact += int((d == 0).sum())
        ulp += int((d == 1).sum())
    assert ulp <= 1e-3 * (exact + ulp)
    # parity frames: the RS code of OUR data frames, bit-exact (oracle)
    m = O.encoding_matrix(50, 75)
    for c in range(AIR_CUBES):
        grp = mine[c * 75:(c + 1) * 75]
        data = [p for *_, p in grp[:50]]
        assert [p for *_, p in grp[50:]] == O.rs_encode(m, 50, data)


def test_queue_depth_does_not_change_stream(P, flight, result):
    from paper_2602_13509_b200.air import run_air

    assert run_air(config(queue_depth=1), flight).frames == result.frames
    assert run_air(config(queue_depth=3), flight).frames == result.frames


def test_timings_and_save_stage(P, flight, tmp_path):
    from paper_2602_13509_b200.air import run_air

    res = run_air(config(out_dir=tmp_path / "raw"), flight)
    assert len(res.timings) == AIR_CUBES
    assert all(v >= 0.0 for t in res.timings for v in t.as_tuple())
    files = sorted((tmp_path / "raw").glob("cube_*.hsc"))
    assert len(files) == AIR_CUBES
    # .hsc ingest: the same flight from the saved files gives the same stream
    paths = SimpleNamespace(cubes=files, tables=flight.tables)
    assert run_air(config(), paths).frames == res.frames


def test_poisoned_cube_dropped_in_isolation(P, flight, result):
    from paper_2602_13509_b200.air import run_air

    bad = flight.cubes[1]
    poison = tuple(dataclasses.replace(m, gain=1e-40) for m in bad.line_meta)
    cubes = list(flight.cubes)
    cubes[1] = P.RawCube(bad.values, bad.wavelengths_nm, poison)
    res = run_air(config(), SimpleNamespace(cubes=cubes, tables=flight.tables))
    assert len(res.dropped) == 1 and res.dropped[0][0] == 1
    assert res.dropped[0][1].startswith("detect: ") and "non-finite" in res.dropped[0][1]
    assert len(res.timings) == AIR_CUBES - 1
    assert {struct.unpack_from("<I", f)[0] // 1 for f in res.frames} == {0, 2}
    assert res.frames[:75] == result.frames[:75] and res.frames[75:] == result.frames[150:]


def test_hsc_round_trip_matches_reference_bytes(P, golden, tmp_path):
    from paper_2602_13509_b200 import formats

    blob = golden["air"]["tiny_hsc"].tobytes()
    path = tmp_path / "t.hsc"
    path.write_bytes(blob)
    cube = formats.read_cube(path)
    assert cube.values.shape == (3, 4, 5)
    assert np.array_equal(cube.values, np.arange(60, dtype=np.uint16).reshape(3, 4, 5) * 7)
    assert [m.gain for m in cube.line_meta] == [1.0, 0.5, 2.0]
    out = tmp_path / "u.hsc"
    formats.write_cube(out, cube)
    assert out.read_bytes() == blob
    dc = formats.read_cube(path, device=True)
    assert dc.values.is_cuda and np.array_equal(dc.values.cpu().numpy(), cube.values)
    from paper_2602_13509_b200.errors import FormatError

    path.write_bytes(blob[:-1])
    with pytest.raises(FormatError, match="truncated payload"):
        formats.read_cube(path)
    path.write_bytes(b"XSC1" + blob[4:])
    with pytest.raises(FormatError, match="bad magic"):
        formats.read_cube(path)
