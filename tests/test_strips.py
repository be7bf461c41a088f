"""Multi-strip sharding (BASELINE config 4) on CPU: world_size 2 over gloo.

paper_2602_13509_b200.strips.detect_strips is the product's partitioning:
strip i -> rank i % world, each rank runs only its strips (no data-path
collective), then an all-gather of the per-strip summaries.  Here the local
work is the CPU oracle behind the same ``ops`` interface (the CUDA ops,
StripBatch, run on the GPU in tests/test_gpu_strips.py).  Every strip must
be processed exactly once, by its owner, with the single-process oracle's
result, and every rank must see the same summary.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import skyrx_oracle as O
from oracle import synth as osynth
from paper_2602_13509_b200.rx import Detection
from paper_2602_13509_b200.strips import detect_strips, shard_strips, strip_owner


class Strip:
    def __init__(self, values):
        self.values = values
        self.lines, self.samples, self.bands = values.shape


def make_source(seed0, L, S, B):
    def source(i):
        t = osynth.make_tables(seed0 + i, S, B, 3)
        return Strip(osynth.generate_lines(t, 0, L)), t
    return source


class OracleStripOps:
    """detect_strips' ops interface with the CPU oracle as the local work."""

    def __init__(self):
        self.seen = []

    def run(self, indices, source, k=None, host=None):
        out = {}
        for i in indices:
            raw, t = source(i)
            self.seen.append(i)
            st, sc, mask = O.detect(raw.values, t.dark, t.coeff, np.ones(raw.lines), k)
            out[i] = Detection(st, sc, mask, O.topk_threshold(sc, k), O.max_score(sc))
        return out


def _worker(rank, world, port, args, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, seed0, L, S, B = args
        ops = OracleStripOps()
        res = detect_strips(make_source(seed0, L, S, B), n, ops=ops)
        q.put((rank, res.world, sorted(res.local), ops.seen,
               [(s.index, s.rank, s.threshold, s.max_score, s.anomalies) for s in res.summary],
               {i: (d.stats.sigma_inv, d.scores, d.mask) for i, d in res.local.items()}))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_round_robin():
    for n in (0, 1, 7, 64):
        for world in (1, 2, 3, 8):
            parts = [shard_strips(n, r, world) for r in range(world)]
            flat = sorted(i for p in parts for i in p)
            assert flat == list(range(n))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1
            assert all(strip_owner(i, world) == r for r, p in enumerate(parts) for i in p)
    with pytest.raises(ValueError):
        shard_strips(4, 2, 2)


@pytest.mark.parametrize("n", [5, 2])
def test_two_rank_strips_equal_single_process(n):
    args = (n, 300, 24, 20, 8)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, args, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((r[0], r[1:]) for r in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # each strip once, by its owner; no rank touched another rank's strip
    for r in (0, 1):
        world, local, seen, summary, res = out[r]
        assert world == 2
        assert local == seen == shard_strips(n, r, 2)
    assert sorted(out[0][1] + out[1][1]) == list(range(n))
    # every rank sees the identical gathered summary of all strips
    assert out[0][3] == out[1][3]
    assert [s[0] for s in out[0][3]] == list(range(n))
    # and the results are the single-process oracle's
    source = make_source(*args[1:])
    for i in range(n):
        r = strip_owner(i, 2)
        sinv, sc, mask = out[r][4][i]
        raw, t = source(i)
        st, want_sc, want_mask = O.detect(raw.values, t.dark, t.coeff, np.ones(raw.lines))
        assert np.array_equal(sinv, st.sigma_inv)
        assert np.array_equal(sc, want_sc) and np.array_equal(mask, want_mask)
        assert out[0][3][i][1] == r
        assert out[0][3][i][4] == int(want_mask.sum())


def test_single_process_is_world_one():
    ops = OracleStripOps()
    res = detect_strips(make_source(300, 24, 20, 8), 3, ops=ops)
    assert res.world == 1 and ops.seen == [0, 1, 2]
    assert [s.index for s in res.summary] == [0, 1, 2]
    with pytest.raises(ValueError, match="n_strips"):
        detect_strips(make_source(300, 24, 20, 8), ops=ops)
