"""Independent flight strips sharded over ranks (BASELINE config 4).

The reference's caller walks cubes one at a time, each with its own background
(`pipeline.py:152-235`: `compute_stats` + `rx_scores` per cube, `rx.py:42-97`).
Strips never share data, so multi-GPU is pure work partitioning: strip i
belongs to rank ``i % world`` (round-robin, so every rank gets ⌊n/world⌋ or
⌈n/world⌉ strips), every rank runs its share through one batched device plan
(moments of all its strips, ONE batched Cholesky/inverse, scores + top-0.1 %
masks), and no collective touches the data path.  The only collective is an
optional all-gather of the per-strip summaries (index, status, threshold,
max score: a few bytes per strip) so every rank can report the whole job.

Layers:
  * :class:`StripBatch` — the device-resident batch of one rank
    (graph-capturable :meth:`enqueue`, then :meth:`verify`: status and flags
    of EVERY slot, general-path redo of any strip the fast kernels could not
    take, the reference's ValueErrors);
  * :func:`detect_strips` — the user call: shard, run, (gather), with the
    local work behind a small ``ops`` interface so the CPU tests drive the
    same sharding with an oracle-backed ops object (tests/test_strips.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np
import torch
import torch.distributed as dist

from . import _dev, _lib
from .calibrate import _check_tables, _raw_device, line_gains, tables_of
from .rx import _STATUS_MSG, DetectPlan, Detection, constant_gain, key_to_float

# score flags that mean "the exact-digit score kernel did not apply to this slot"
# (include/skyrx_b200.h: 16 counts >= 4096, 32 no no-clamp proof); moments that must
# be redone are _lib.flags_range (2 quantiser range, 4 clamp not corrected by 256)
RESCORE_FLAGS = 16 | 32


def needs_redo(flags: int) -> bool:
    return _lib.flags_range(flags) or bool(int(flags) & RESCORE_FLAGS)


def strip_owner(index: int, world: int) -> int:
    """Rank that processes strip ``index`` (round-robin)."""
    return index % world


def shard_strips(n_strips: int, rank: int, world: int) -> list[int]:
    """Global indices of the strips rank ``rank`` of ``world`` processes."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    return list(range(rank, n_strips, world))


def rank_world(group=None) -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


@dataclass
class StripSummary:
    """Per-strip outcome every rank can see after the gather (a few bytes)."""

    index: int
    rank: int
    status: int
    threshold: float
    max_score: float
    anomalies: int
    redone: bool = False


@dataclass
class StripsResult:
    local: dict                      # global index -> Detection (this rank's strips)
    summary: list = field(default_factory=list)   # StripSummary of every strip (gathered)
    rank: int = 0
    world: int = 1


class StripBatch:
    """One rank's strips of one shape, resident on the device.

    ``raws[j]`` are device u16 (L, S, B) tensors, ``tables[j]`` device
    (dark, coeff) pairs, ``gains[j]`` device f32 (L,) and ``gain_const[j]`` the
    common line gain or None (``rx.constant_gain``).  :meth:`enqueue` issues
    every kernel of every strip with no host synchronisation (what bench.py
    captures in one CUDA graph); :meth:`verify` is the host check after it.
    """

    def __init__(self, lines: int, samples: int, bands: int, count: int):
        if count < 1:
            raise ValueError("a strip batch needs at least one strip")
        self.shape = (lines, samples, bands)
        self.count = count
        self.plan = DetectPlan(lines, samples, bands, batch=count)

    @property
    def launches(self) -> int:
        return self.plan.launches

    def enqueue(self, raws, tables, gains, gain_const, k: int | None = None,
                moment_events=None, score_events=None):
        """Moments of every strip -> one batched finalize -> scores + masks.

        ``moment_events[j]`` / ``score_events[j]`` = optional (start, end) CUDA
        event pairs recorded around strip j's moments / score kernel alone."""
        plan = self.plan
        for j in range(self.count):
            d, c = tables[j]
            plan.run(j, raws[j], d, c, gains[j], gain_const=gain_const[j],
                     events=None if moment_events is None else moment_events[j])
        plan.finalize()
        for j in range(self.count):
            d, c = tables[j]
            plan.score(j, raws[j], d, c, gains[j], k,
                       events=None if score_events is None else score_events[j])
        return self

    def flags(self) -> tuple[np.ndarray, np.ndarray]:
        """(status, flags) of every slot (one small D2H each)."""
        return self.plan.ds.status.cpu().numpy(), self.plan.ds.flags.cpu().numpy()

    def verify(self, raws, tables, gains, k: int | None = None) -> list[int]:
        """Check EVERY slot after :meth:`enqueue`: redo (synchronously, general
        kernels) any strip whose fast path did not apply, then raise the
        reference's ValueError for a strip that still failed.  Returns the
        redone slots."""
        cubes = {j: (raws[j], tables[j][0], tables[j][1], gains[j]) for j in range(self.count)}
        redone = self.plan.recover_range(cubes)
        st, fl = self.flags()
        bad = [j for j in range(self.count) if needs_redo(fl[j]) and j not in redone]
        if bad:
            # a slot still flagged after recover_range: the general kernels again
            for j in bad:
                self.plan.run(j, *cubes[j], force_ffma=True)
                self.plan.finalize(j)
                keep = (self.plan.tcw, self.plan.tcs)
                self.plan.tcw = self.plan.tcs = False
                self.plan.used_raw[j] = False
                self.plan.score(j, *cubes[j], k)
                self.plan.tcw, self.plan.tcs = keep
            redone = sorted(set(redone) | set(bad))
            st, fl = self.flags()
        L, S, B = self.shape
        for j in range(self.count):
            if st[j] == _lib.ERR_INSUFFICIENT:
                raise ValueError(f"insufficient samples: {L * S} pixels for {B} bands")
            if st[j] != _lib.OK:
                raise ValueError(_STATUS_MSG.get(int(st[j]), f"stats failed with status {st[j]}"))
        return redone

    def detection(self, j: int, host: bool = False) -> Detection:
        plan = self.plan
        L, S, _ = self.shape
        stats = plan.ds.host(j, L * S)
        thr = float(plan.thr[j].item())
        mx = key_to_float(plan.max_key[j])
        if host:
            return Detection(stats, _dev.to_host(plan.scores[j]),
                             _dev.to_host(plan.mask[j]).view(bool), thr, mx)
        return Detection(stats, plan.scores[j], plan.mask[j].view(torch.bool), thr, mx)


class CudaStripOps:
    """Local work of :func:`detect_strips` on this rank's GPU (the product path)."""

    def run(self, indices: Sequence[int], source: Callable, k: int | None = None,
            host: bool | None = None) -> dict:
        if not indices:
            return {}
        cubes = [source(i) for i in indices]
        raw0 = cubes[0][0]
        L, S, B = raw0.lines, raw0.samples, raw0.bands
        raws, tabs, gains, gconst = [], [], [], []
        for raw, tab in cubes:
            if (raw.lines, raw.samples, raw.bands) != (L, S, B):
                raise ValueError("detect_strips: every strip must have the same shape")
            if raw.lines * raw.samples <= raw.bands:
                raise ValueError(f"insufficient samples: {raw.lines * raw.samples} pixels "
                                 f"for {raw.bands} bands")
            tab = tables_of(tab)
            _check_tables(raw, tab)
            g = line_gains(raw)
            raws.append(_raw_device(raw))
            tabs.append(tab.device())
            gains.append(_dev.to_device(g, torch.float32))
            gconst.append(constant_gain(g, tab))
        batch = StripBatch(L, S, B, len(indices))
        batch.enqueue(raws, tabs, gains, gconst, k)
        batch.verify(raws, tabs, gains, k)
        out = {}
        for j, (i, (raw, _)) in enumerate(zip(indices, cubes)):
            on_host = (not _dev.is_device(raw.values)) if host is None else host
            out[i] = batch.detection(j, host=on_host)
        return out


def detect_strips(source, n_strips: int | None = None, *, k: int | None = None, group=None,
                  ops=None, gather: bool = True, host: bool | None = None) -> StripsResult:
    """Detect every strip of a multi-strip job, sharded over the ranks of ``group``.

    ``source`` is a sequence of (RawCube, CalibrationTables) pairs or a callable
    ``source(i) -> (RawCube, CalibrationTables)`` (so a rank only materialises
    its own strips); ``n_strips`` is required for a callable.  Each rank
    processes strips ``shard_strips(n, rank, world)`` with no data-path
    collective and returns their detections in ``local``; with ``gather`` the
    per-strip :class:`StripSummary` of every strip is all-gathered (control
    plane only).  Single process (no process group): world = 1, every strip.
    """
    if callable(source):
        if n_strips is None:
            raise ValueError("detect_strips: n_strips is required with a callable source")
        get = source
    else:
        seq = list(source)
        n_strips = len(seq) if n_strips is None else n_strips
        get = seq.__getitem__
    rank, world = rank_world(group)
    mine = shard_strips(n_strips, rank, world)
    ops = ops or CudaStripOps()
    local = ops.run(mine, get, k=k, host=host)
    summ = [StripSummary(i, rank, _lib.OK, float(d.threshold), float(d.max_score),
                         _count(d.mask)) for i, d in local.items()]
    if gather and world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, summ, group=group)
        summ = [s for p in parts for s in p]
    summ.sort(key=lambda s: s.index)
    return StripsResult(local=local, summary=summ, rank=rank, world=world)


def _count(mask) -> int:
    if isinstance(mask, torch.Tensor):
        return int(torch.count_nonzero(mask).item())
    return int(np.count_nonzero(mask))
