"""GF(256) erasure code + frames on the GPU, bit-exact against the
reference's outputs (tests/golden/fec.npz) and the oracle; cases follow the reference's
tests/test_fec.py."""

import dataclasses

import numpy as np
import pytest

from oracle import skyrx_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    from paper_2602_13509_b200 import build, fec

    build.build()
    return fec


@pytest.fixture(scope="module")
def code(F):
    return F.ErasureCode(50, 25)


def test_matmul_matches_reference(F, golden):
    g = golden["fec"]
    assert np.array_equal(F.gf256_matmul(g["mm/mat"], g["mm/data"]), g["mm/out"])


@pytest.mark.parametrize("r,k,n,seed", [(1, 1, 1, 0), (25, 50, 3728, 1), (9, 13, 7, 2),
                                        (256, 256, 1031, 3), (3, 200, 20000, 4), (17, 5, 8, 5)])
def test_matmul_matches_oracle(F, r, k, n, seed):
    rng = np.random.default_rng(seed)
    mat = rng.integers(0, 256, (r, k), dtype=np.uint8)
    data = rng.integers(0, 256, (k, n), dtype=np.uint8)
    data[:, ::5] = 0
    assert np.array_equal(F.gf256_matmul(mat, data), O.gf256_matmul(mat, data))


def test_device_in_device_out(F):
    import torch

    rng = np.random.default_rng(9)
    mat = rng.integers(0, 256, (4, 6), dtype=np.uint8)
    data = rng.integers(0, 256, (6, 100), dtype=np.uint8)
    out = F.gf256_matmul(torch.from_numpy(mat).cuda(), torch.from_numpy(data).cuda())
    assert out.is_cuda and np.array_equal(out.cpu().numpy(), O.gf256_matmul(mat, data))


def test_inverse(F, golden):
    g = golden["fec"]
    assert np.array_equal(F.gf_mat_inv(g["inv/m"]), g["inv/minv"])
    with pytest.raises(np.linalg.LinAlgError, match="singular"):
        F.gf_mat_inv(np.array([[1, 2], [1, 2]], np.uint8))
    rng = np.random.default_rng(4)
    for k in (1, 2, 37, 128, 256):
        m = rng.integers(0, 256, (k, k), dtype=np.uint8)
        try:
            want = O.gf_mat_inv(m)
        except np.linalg.LinAlgError:
            with pytest.raises(np.linalg.LinAlgError):
                F.gf_mat_inv(m)
            continue
        assert np.array_equal(F.gf_mat_inv(m), want), k


@pytest.mark.parametrize("k,p", [(50, 25), (4, 3), (1, 0), (200, 56)])
def test_encoding_matrix_matches_reference(F, golden, k, p):
    assert np.array_equal(F.ErasureCode(k, p).matrix, golden["fec"][f"matrix_{k}_{p}"])


def test_encode_decode_match_reference(F, code, golden):
    g = golden["fec"]
    coded = [r.tobytes() for r in g["enc/coded"]]
    assert code.encode(coded[:50]) == coded[50:]
    cases, c = [], 0
    while f"dec{c}/keep" in g:
        cases.append([(int(i), coded[i]) for i in g[f"dec{c}/keep"]])
        c += 1
    batch = code.decode_groups(cases)
    for c, received in enumerate(cases):
        for out, rep in (code.decode(received), batch[c]):
            assert sorted(out) == g[f"dec{c}/slots"].tolist()
            assert b"".join(out[i] for i in sorted(out)) == g[f"dec{c}/data"].tobytes()
            assert list(rep.recovered) == g[f"dec{c}/recovered"].tolist()
            assert list(rep.missing) == g[f"dec{c}/missing"].tolist()
            assert len(rep.received) == g[f"dec{c}/report"][0]


def test_reference_fec_behaviours(F, code):
    from paper_2602_13509_b200.errors import ProtocolError

    assert np.array_equal(code.matrix[:50], np.eye(50, dtype=np.uint8))
    assert all(p == bytes(64) for p in code.encode([bytes(64)] * 50))
    with pytest.raises(ValueError, match="50"):
        code.encode([bytes(8)] * 49)
    with pytest.raises(ValueError, match="length"):
        code.encode([bytes(8)] * 49 + [bytes(9)])
    rng = np.random.default_rng(77)
    payloads = [rng.integers(0, 256, 211, dtype=np.uint8).tobytes() for _ in range(50)]
    frames = list(enumerate(payloads + code.encode(payloads)))
    with pytest.raises(ProtocolError, match="duplicate"):
        code.decode(frames + [frames[3]])
    rec, rep = code.decode([])
    assert rec == {} and rep.missing == tuple(range(50))
    for _ in range(10):
        keep = sorted(rng.permutation(75)[:50])
        rec, rep = code.decode([frames[i] for i in keep])
        assert rep.complete and [rec[i] for i in range(50)] == payloads
    small = F.ErasureCode(4, 3)
    data = [b"abcd", b"efgh", b"ijkl", b"mnop"]
    coded = list(enumerate(data + small.encode(data)))
    for drop in ([0, 1, 2], [0, 2, 4], [4, 5, 6], [1, 3, 5]):
        rec, rep = small.decode([f for f in coded if f[0] not in drop])
        assert rep.complete and [rec[i] for i in range(4)] == data


def test_frames_match_reference(golden):
    from paper_2602_13509_b200 import datalink as D

    g = golden["fec"]
    pk = [r.tobytes() for r in g["frames/packets"].reshape(100, -1)]
    frames = D.frames_for_cube(3, pk)
    assert [len(f) for f in frames] == g["frames/lengths"].tolist()
    assert b"".join(frames) == g["frames/frames"].tobytes()
    assert D.parse_frame(frames[60])[:3] == (6, 60, 1)
    with pytest.raises(ValueError, match="multiple"):
        D.frames_for_cube(0, pk[:49])


@pytest.mark.parametrize("lines", [50, 1000])
def test_cube_frames_fused(lines):
    import paper_2602_13509_b200 as P
    from paper_2602_13509_b200 import datalink as D

    rng = np.random.default_rng(lines)
    rgb = (rng.random((lines, 900, 3)) * 30).astype(np.float32)
    sc = (rng.random((lines, 900)) ** 4 * 900).astype(np.float32)
    ins = P.InsSample(5, 35.0, -90.0, 40.0, 0.0, 0.0, 0.0)
    metas = [P.LineMeta(1000 + i, 1.0, ins, ins) for i in range(lines)]
    pk = D.packetize_cube(2, rgb, sc, metas)
    fr = D.cube_frames(2, rgb, sc, metas)
    assert fr == D.frames_for_cube(2, pk)
    t = dataclasses.astuple(ins)
    om = [(m.exposure_start_us, t, t) for m in metas]
    opk = O.packetize_cube(2, rgb, sc, om)
    assert pk == opk
    if lines == 50:
        assert fr == O.frames_for_cube(2, opk)
