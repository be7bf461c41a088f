"""GF(256) Reed-Solomon erasure code of the downlink on the device.

Drop-in for skyrx.fec (fec.py:28-195) and `_accel.gf256_matmul` (_accel.py:50-70,
92-107): parity generation and erasure recovery are GF(2^8) matrix products over the
payload bytes, done by `skyrx_gf_matmul` (csrc/fec.cu, bit-sliced, no table lookups);
the k x k inverse of an erasure pattern by `skyrx_gf_invert` (one CTA per group, the
reference's Gauss-Jordan pivot rule). Scalar field helpers (gf_mul / gf_inv / gf_pow) stay
on the host, as in the reference, for building the Vandermonde matrix.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np
import torch

from . import _dev, _lib, errors

GF_PRIM = 0x11D               # fec.py:28-29
GF_GEN = 2
GROUP_DATA = 50               # fec.py:32-33: the link's 50 data + 25 parity frames
GROUP_PARITY = 25


def _tables():
    exp = np.zeros(510, np.uint8)
    log = np.zeros(256, np.int16)
    v = 1
    for e in range(255):
        exp[e] = exp[e + 255] = v
        log[v] = e
        v = ((v << 1) ^ GF_PRIM) if v & 0x80 else (v << 1)
    return log, exp


GF_LOG, GF_EXP = _tables()


def gf_mul(a: int, b: int) -> int:
    return 0 if a == 0 or b == 0 else int(GF_EXP[int(GF_LOG[a]) + int(GF_LOG[b])])


def gf_inv(a: int) -> int:
    if a == 0:
        raise ZeroDivisionError("no inverse of 0 in GF(256)")
    return int(GF_EXP[255 - int(GF_LOG[a])])


def gf_pow(x: int, n: int) -> int:
    """fec.py:65-70, keeping its int16 product: log[x] * n wraps past 32767 (NEP 50)."""
    if n == 0:
        return 1
    if x == 0:
        return 0
    e = (int(GF_LOG[x]) * n + 32768) % 65536 - 32768
    return int(GF_EXP[e % 255])


def _u8(x) -> torch.Tensor:
    return _dev.to_device(x, torch.uint8).contiguous()


def _matmul_dev(mat: torch.Tensor, data: torch.Tensor) -> torch.Tensor:
    r, k = mat.shape
    n = data.shape[1]
    out = _dev.empty((r, n), torch.uint8)
    _lib.call("skyrx_gf_matmul", mat.data_ptr(), 0, r, k, data.data_ptr(), n, 0, n,
              out.data_ptr(), n, 0, 1, _dev.stream_ptr())
    return out


def gf256_matmul(mat, data, gf_log=None, gf_exp=None):
    """`mat @ data` over GF(256) (_accel.py:50-70): (r, k) u8 times (k, n) u8.  The tables
    arguments are accepted for signature parity; the field is fixed (poly 0x11D).  Device
    tensors in -> device tensor out; numpy in -> numpy out."""
    m, d = _u8(mat), _u8(data)
    if m.dim() != 2 or d.dim() != 2 or m.shape[1] != d.shape[0]:
        raise ValueError(f"shape mismatch: {tuple(m.shape)} @ {tuple(d.shape)}")
    if m.shape[0] == 0 or d.shape[1] == 0:
        out = _dev.zeros((m.shape[0], d.shape[1]), torch.uint8)
    else:
        out = _matmul_dev(m, d)
    return _dev.like_input(data, out)


def _invert_rows(mat_d: torch.Tensor, rows: np.ndarray, sel: np.ndarray, nsel: np.ndarray):
    """Batched: per problem g, rows sel[g, :nsel[g]] of inv(mat[rows[g]]) (k x k, zero padded)."""
    g, k = rows.shape
    out = _dev.empty((g, k, k), torch.uint8)
    status = _dev.empty((g,), torch.int32)
    rd, sd = _dev.to_device(rows.astype(np.int32)), _dev.to_device(sel.astype(np.int32))
    nd = _dev.to_device(nsel.astype(np.int32))
    _lib.call("skyrx_gf_invert", mat_d.data_ptr(), mat_d.shape[1], rd.data_ptr(), k, sd.data_ptr(),
              nd.data_ptr(), g, out.data_ptr(), status.data_ptr(), _dev.stream_ptr())
    return out, status


def gf_mat_inv(m) -> np.ndarray:
    """Inverse of a square GF(256) matrix (fec.py:82-98)."""
    m = np.asarray(m, np.uint8)
    k = m.shape[0]
    if m.shape != (k, k) or k == 0:
        raise ValueError("square matrix required")
    idx = np.arange(k)[None, :]
    inv, status = _invert_rows(_u8(m), idx, idx, np.array([k]))
    if int(status.item()):
        raise np.linalg.LinAlgError("singular matrix over GF(256)")
    return _dev.to_host(inv[0])


@dataclass(frozen=True)
class FecReport:
    """fec.py:117-125: outcome of decoding one group, in data-slot indices (0..k-1)."""

    received: tuple
    recovered: tuple
    missing: tuple

    @property
    def complete(self) -> bool:
        return not self.missing


class ErasureCode:
    """Reed-Solomon erasure codec for fixed (data, parity) counts (fec.py:128-195)."""

    def __init__(self, data_count: int = GROUP_DATA, parity_count: int = GROUP_PARITY):
        if data_count < 1 or parity_count < 0:
            raise ValueError("counts must be positive")
        total = data_count + parity_count
        if total > 256:
            raise ValueError("at most 256 coded payloads in GF(256)")
        self.data_count, self.parity_count, self.total = data_count, parity_count, total
        # fec.py:101-115: Vandermonde at points 0..total-1, made systematic by inv(V[:k])
        vand = np.array([[gf_pow(i, j) for j in range(data_count)] for i in range(total)],
                        np.uint8)
        vd = _u8(vand)
        idx = np.arange(data_count)[None, :]
        top_inv, status = _invert_rows(vd, idx, idx, np.array([data_count]))
        if int(status.item()):
            raise np.linalg.LinAlgError("singular matrix over GF(256)")
        self._matrix_d = _matmul_dev(vd, top_inv[0])
        self._parity_d = self._matrix_d[data_count:].contiguous()
        self.matrix = _dev.to_host(self._matrix_d)

    # ---------------------------------------------------------------- encode
    def encode_groups(self, data: torch.Tensor, pitch: int | None = None,
                      out: torch.Tensor | None = None) -> torch.Tensor:
        """Parity of G groups at once on the device: `data` is (G, k, n) u8 (or rows of
        `pitch` bytes, k consecutive rows per group) -> (G, parity, n) u8."""
        g, k, n = data.shape
        if k != self.data_count:
            raise ValueError(f"invalid group: expected {self.data_count} payloads, got {k}")
        p = self.parity_count
        if out is None:
            out = _dev.empty((g, p, n), torch.uint8)
        if p and n and g:
            dp = pitch if pitch is not None else n
            _lib.call("skyrx_gf_matmul", self._parity_d.data_ptr(), 0, p, k, data.data_ptr(), dp,
                      k * dp, n, out.data_ptr(), n, p * n, g, _dev.stream_ptr())
        return out

    def encode(self, payloads: Sequence[bytes]) -> list[bytes]:
        """fec.py:140-155: parity payloads for exactly data_count equal-length payloads."""
        if len(payloads) != self.data_count:
            raise ValueError(
                f"invalid group: expected {self.data_count} payloads, got {len(payloads)}")
        length = len(payloads[0])
        if any(len(p) != length for p in payloads):
            raise ValueError("invalid group: payload lengths differ")
        if self.parity_count == 0:
            return []
        data = _u8(np.frombuffer(b"".join(payloads), np.uint8).reshape(1, self.data_count,
                                                                        length))
        par = _dev.to_host(self.encode_groups(data)[0])
        return [par[i].tobytes() for i in range(self.parity_count)]

    # ---------------------------------------------------------------- decode
    def decode(self, received: Iterable[tuple[int, bytes]]):
        """fec.py:157-195: recover data payloads from any subset of coded payloads."""
        plan = self._plan(received)
        if plan[0] is not None:
            return plan[0]
        out, entries, absent, direct = plan[1:]
        rec = self._recover([(entries, absent)])[0]
        for slot, row in zip(absent, rec):
            out[slot] = row.tobytes()
        return out, FecReport(received=direct, recovered=absent, missing=())

    def decode_groups(self, groups: Sequence[Iterable[tuple[int, bytes]]]):
        """decode() over many groups with one inverse launch and one matmul launch for all
        groups that need recovery (the ground side's per-cube batch)."""
        results, todo = [None] * len(groups), []
        for gi, received in enumerate(groups):
            plan = self._plan(received)
            if plan[0] is not None:
                results[gi] = plan[0]
            else:
                todo.append((gi, plan[1:]))
        if todo:
            recs = self._recover([(p[1], p[2]) for _, p in todo])
            for (gi, (out, _, absent, direct)), rec in zip(todo, recs):
                for slot, row in zip(absent, rec):
                    out[slot] = row.tobytes()
                results[gi] = (out, FecReport(received=direct, recovered=absent, missing=()))
        return results

    def _plan(self, received):
        entries = sorted(received, key=lambda e: e[0])
        indices = [i for i, _ in entries]
        if len(set(indices)) != len(indices):
            raise errors.ProtocolError("duplicate coded index in group")
        if indices and (indices[0] < 0 or indices[-1] >= self.total):
            raise errors.ProtocolError(f"coded index outside 0..{self.total - 1}")
        if len({len(p) for _, p in entries}) > 1:
            raise errors.ProtocolError("received payload lengths differ")
        out = {i: p for i, p in entries if i < self.data_count}
        direct = tuple(sorted(out))
        absent = tuple(i for i in range(self.data_count) if i not in out)
        if len(entries) < self.data_count or not absent:
            return (out, FecReport(received=direct, recovered=(), missing=absent)),
        return None, out, entries[: self.data_count], absent, direct

    def _recover(self, problems):
        """[(chosen k entries, absent slots)] -> recovered rows per problem (numpy)."""
        k = self.data_count
        g = len(problems)
        lengths = {len(e[0][1]) for e, _ in problems}
        rows = np.array([[i for i, _ in e] for e, _ in problems], np.int64)
        sel = np.zeros((g, k), np.int64)
        nsel = np.array([len(a) for _, a in problems], np.int64)
        for i, (_, a) in enumerate(problems):
            sel[i, : len(a)] = a
        inv, status = _invert_rows(self._matrix_d, rows, sel, nsel)
        r = int(nsel.max())
        outs = []
        for length in sorted(lengths):   # one launch per payload length (normally one)
            ids = [i for i, (e, _) in enumerate(problems) if len(e[0][1]) == length]
            stacked = np.frombuffer(b"".join(p for i in ids for _, p in problems[i][0]),
                                    np.uint8).reshape(len(ids), k, length)
            sd = _u8(stacked)
            mats = inv[torch.as_tensor(ids, device=inv.device)] if len(ids) != g else inv
            res = _dev.empty((len(ids), r, length), torch.uint8)
            if length:
                _lib.call("skyrx_gf_matmul", mats.data_ptr(), k * k, r, k, sd.data_ptr(), length,
                          k * length, length, res.data_ptr(), length, r * length, len(ids),
                          _dev.stream_ptr())
            else:
                res.zero_()
            outs.append((ids, _dev.to_host(res)))
        if int(status.max().item()):
            raise np.linalg.LinAlgError("singular matrix over GF(256)")
        result = [None] * g
        for ids, res in outs:
            for j, i in enumerate(ids):
                result[i] = res[j, : nsel[i]]
        return result
