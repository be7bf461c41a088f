"""Link payload epilogue on the GPU: bit-exact against the
reference's own outputs (tests/golden/datalink.npz) and the CPU oracle."""

import numpy as np
import pytest

from oracle import skyrx_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def D():
    from paper_2602_13509_b200 import build, datalink

    build.build()
    return datalink


def test_row_encodings_match_reference(D, golden):
    g = golden["datalink"]
    assert np.array_equal(D.pack_rgb565(g["row/rgb"], 40.0, 37.5, 12.25), g["row/rgb565"])
    assert np.array_equal(D.encode_scores_half(g["row/scores"], 500.0), g["row/half"])
    assert np.array_equal(D.encode_scores_half(g["row/scores"], 0.0), g["row/half_zero_max"])
    assert np.array_equal(D.pack_rgb565(g["row/rgb"], 0.0, 37.5, -1.0), g["row/rgb565_zero_max"])


def test_packetize_cube_matches_reference(D, golden):
    import paper_2602_13509_b200 as P

    g = golden["datalink"]
    lines = g["cube/rgb"].shape[0]
    metas = []
    for i in range(lines):  # tests/golden/make_golden.py metas()
        t = 1_600_000_000_000_000 + i * 4016
        metas.append(P.LineMeta(t, 1.0, P.InsSample(t - 1000, 35.0, -90.0, 40.0, 0.0, 0.0, 0.0),
                                P.InsSample(t + 4000, 35.0, -90.0, 40.0, 0.0, 0.0, 0.0)))
    pk = D.packetize_cube(7, g["cube/rgb"], g["cube/scores"], metas)
    assert np.array_equal(np.frombuffer(b"".join(pk), np.uint8), g["cube/packets"])


@pytest.mark.parametrize("lines,samples,seed", [(64, 900, 1), (5, 37, 2), (1, 1, 3)])
def test_whole_cube_payload_matches_oracle(D, lines, samples, seed):
    rng = np.random.default_rng(seed)
    rgb = (rng.random((lines, samples, 3)) * 30).astype(np.float32)
    sc = (rng.random((lines, samples)) ** 5 * 1e3).astype(np.float32)
    words, (ms, mr, mg, mb) = D.link_payload(rgb, sc)
    w = words.cpu().numpy()
    assert (ms, mr, mg, mb) == (float(sc.max()), float(rgb[..., 0].max()),
                                float(rgb[..., 1].max()), float(rgb[..., 2].max()))
    assert np.array_equal(w[..., 0], O.pack_rgb565(rgb, mr, mg, mb))
    assert np.array_equal(w[..., 1], O.encode_scores_half(sc, ms))
