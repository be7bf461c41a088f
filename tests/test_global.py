"""R-GLOBAL protocol (BASELINE config 5) on CPU: world_size 2 over gloo.

paper_2602_13509_b200.distributed.global_detect is the product's exchange
logic (shift broadcast, FP64 moment SUM all-reduce, non-finite MAX, global
max, 3-round radix-histogram all-reduce for the top-0.1 % threshold).  Here
it runs on two CPU processes with an ops object whose local work is the CPU
oracle (the CUDA ops are covered on the GPU by tests/test_gpu_global.py).
The result must equal the single-process oracle on the concatenated cube.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import skyrx_oracle as O
from oracle import synth as osynth

HIST_BINS = 2048


def f2ord(v):
    u = np.asarray(v, np.float32).view(np.uint32).astype(np.uint64)
    return np.where(u & 0x80000000, ~u & 0xFFFFFFFF, u | 0x80000000).astype(np.uint64)


def ord2f(u):
    u = int(u)
    b = (u & 0x7FFFFFFF) if (u & 0x80000000) else (~u & 0xFFFFFFFF)
    return float(np.array([b], np.uint32).view(np.float32)[0])


def digit_params(d):
    return [(21, 11), (10, 11), (0, 10)][d]


class OracleOps:
    """The ops interface of distributed.global_detect with CPU-oracle local work."""

    def __init__(self, raw, t, gains=None):
        gains = np.ones(raw.shape[0]) if gains is None else gains
        self.rad = O.apply_calibration(raw, t.dark, t.coeff, gains)
        self.B = raw.shape[2]

    def shift(self, raw):
        return torch.from_numpy(self.rad.reshape(-1, self.B)[:4096].astype(np.float64).mean(0))

    def moments(self, raw, shift):
        n, s, q = O.moments(self.rad, shift.numpy())
        fin = int(not np.isfinite(self.rad).all())
        return torch.from_numpy(np.concatenate([[n], s, q.ravel()])), torch.tensor([fin],
                                                                                   dtype=torch.int32)

    def finalize(self, moments, shift, nonfinite):
        m = moments.numpy()
        return (m, shift.numpy(), int(nonfinite[0]))

    def check(self, h, n_total):
        m, shift, fin = h
        if fin:
            raise ValueError("invalid data: cube contains non-finite values")
        B = self.B
        self.stats = O.finalize_moments(m[0], m[1:1 + B], m[1 + B:].reshape(B, B), shift, B)
        return self.stats

    def score(self, raw):
        sc = O.rx_scores(self.rad, self.stats)
        return torch.from_numpy(sc), torch.tensor([int(f2ord(sc.max()))], dtype=torch.int64)

    def topk_init(self, n, k):
        self.prefix, self.rank, self.all = 0, k + 1, k >= n

    def topk_hist(self, scores, digit):
        h = np.zeros(HIST_BINS, np.int64)
        if not self.all:
            shift, bits = digit_params(digit)
            keys = f2ord(scores.numpy().ravel())
            hi = shift + bits
            sel = keys if hi >= 32 else keys[(keys >> hi) == self.prefix]
            h[: 1 << bits] = np.bincount(((sel >> shift) & ((1 << bits) - 1)).astype(np.int64),
                                         minlength=1 << bits)
        self.hist = torch.from_numpy(h.astype(np.int32))
        return self.hist

    def topk_pick(self, digit):
        if self.all:
            return
        shift, bits = digit_params(digit)
        cnt = self.hist.numpy().astype(np.int64)
        cum, b = 0, (1 << bits) - 1
        while b > 0 and cum + cnt[b] < self.rank:
            cum += cnt[b]
            b -= 1
        self.rank -= cum
        self.prefix = (self.prefix << bits) | b

    def threshold(self):
        return float("-inf") if self.all else ord2f(self.prefix)

    def mask(self, scores):
        return scores > np.float32(self.threshold())

    key_to_float = staticmethod(lambda k: ord2f(int(k)))


def _worker(rank, world, port, args, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_13509_b200.distributed import global_detect

        seed, L, S, B, k = args
        t = osynth.make_tables(seed, S, B, 5)
        per = L // world
        raw = osynth.generate_lines(t, rank * per, per)
        res = global_detect(raw, OracleOps(raw, t), n_total=L * S, k=k)
        q.put((rank, res.stats.mu, res.stats.sigma, res.stats.sigma_inv, res.threshold,
               res.max_score, res.scores.numpy(), np.asarray(res.mask)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("args", [(5, 64, 40, 16, None), (11, 40, 48, 24, 3), (6, 32, 20, 8, 10 ** 6)])
def test_two_rank_global_equals_single_process(args):
    seed, L, S, B, k = args
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
    # every rank holds the identical global background
    for a, b in zip(out[0][:3], out[1][:3]):
        assert np.array_equal(a, b)
    mu, sigma, sinv, thr, mx = out[0][:5]
    t = osynth.make_tables(seed, S, B, 5)
    raw = osynth.generate_lines(t, 0, L)
    rad = O.apply_calibration(raw, t.dark, t.coeff, np.ones(L))
    want = O.compute_stats(rad)
    assert np.abs(mu - want.mu).max() <= 1e-12 * np.abs(want.mu).max()
    assert np.abs(sigma - want.sigma).max() <= 1e-10 * np.abs(want.sigma).max()
    # with the exchanged stats, threshold / max / masks equal the one-process select
    scores = np.concatenate([out[0][5], out[1][5]])
    assert thr == O.topk_threshold(scores, k)
    assert mx == float(scores.max())
    assert np.array_equal(np.concatenate([out[0][6], out[1][6]]), O.topk_mask(scores, k))
