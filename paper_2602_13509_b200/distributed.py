"""R-GLOBAL: one background over line blocks spread across ranks (BASELINE config 5).

SURVEY.md §8(e): the 131072 x 2048 x 128 mosaic is cut into contiguous line
blocks, one per rank (one process per GPU).  The background is the SAME for
every pixel, so the only exchange steps are:

  1. broadcast the moment shift c (B f64) from rank 0's block;
  2. all-reduce SUM of the FP64 moments [n, s = sum(x-c), Q = sum((x-c)(x-c)^T)]
     (1 + B + B^2 doubles, 132 KB at B = 128) and MAX of the status flags;
     every rank then finalizes identical bytes -> identical Cholesky, W, Sigma^-1;
  3. all-reduce MAX of the block's max score (normalize_scores, rx.py:100-105);
  4. the global top-0.1 % threshold: 3 rounds of a SUM all-reduce of the
     2048-bin radix histogram of the local scores (skyrx_topk_hist /
     skyrx_topk_pick), then shard-local masks.

Equal to the single-process oracle on the concatenated cube up to FP64
rounding of the moment sums (threshold and mask exactly, given equal scores).
The protocol is written once against a small `ops` interface: `CudaOps`
(this library's kernels, NCCL over NVLink) is the product; the CPU gloo tests
drive the same protocol with an oracle-backed ops object (tests/test_global.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _dev, _lib
from .calibrate import tables_of
from .rx import DetectPlan, constant_gain, key_to_float, topk_count


@dataclass
class GlobalDetection:
    stats: object        # CubeStats of the GLOBAL background (host, identical on all ranks)
    scores: object       # this rank's block (lines_local, samples) f32 (device tensor)
    mask: object         # this rank's block, bool, top 0.1 % of the WHOLE mosaic
    threshold: float     # global delta_(k+1)
    max_score: float     # global max delta
    n_total: int


class CudaOps:
    """Per-rank device work of the global protocol (the product path)."""

    def __init__(self, lines: int, samples: int, bands: int, tables):
        self.tables = tables_of(tables)
        self.plan = DetectPlan(lines, samples, bands)
        self.shape = (lines, samples, bands)
        self.dark, self.coeff = self.tables.device()
        self.gains = _dev.zeros((lines,), torch.float32) + 1.0
        self.gain_const = 1.0
        self.hist_len = int(_lib.load().skyrx_topk_hist_len())

    def set_gains(self, gains):
        if gains is None:
            self.gains.fill_(1.0)
            self.gain_const = 1.0
        else:
            g = gains if isinstance(gains, torch.Tensor) else torch.from_numpy(
                np.asarray(gains, np.float32))
            self.gains.copy_(g)
            self.gain_const = constant_gain(gains, self.tables)

    def _args(self, raw):
        L, S, B = self.shape
        return (raw.data_ptr(), L, S, B, self.dark.data_ptr(), self.coeff.data_ptr(),
                self.gains.data_ptr())

    def shift(self, raw) -> torch.Tensor:
        ds = self.plan.ds
        _lib.call("skyrx_stats_shift", _lib.IN_RAW_U16, *self._args(raw), ds.shift[0].data_ptr(),
                  _dev.stream_ptr())
        return ds.shift[0]

    def moments(self, raw, shift: torch.Tensor):
        """Local moments about the common shift, and this block's non-finite flag.

        A tensor-core path that could not represent this block (quantiser range /
        an uncorrected clamp at 0, _lib.flags_range) is redone locally in the FFMA kernel BEFORE the
        exchange, so only the non-finite bit is global."""
        plan = self.plan
        ds = plan.ds
        ds.shift[0].copy_(shift)
        plan.run_moments(0, raw, self.dark, self.coeff, self.gains, gain_const=self.gain_const)
        if _lib.flags_range(int(ds.flags[0].item())):
            plan.run_moments(0, raw, self.dark, self.coeff, self.gains, force_ffma=True)
        return ds.moments[0], ds.flags[0:1] & 1

    def finalize(self, moments, shift, nonfinite):
        ds = self.plan.ds
        ds.flags[0:1].bitwise_or_(nonfinite)
        self.plan.finalize()
        return ds

    def check(self, stats, n_total: int):
        stats.check(0, n_total)
        return stats.host(0, n_total)

    def score(self, raw):
        plan = self.plan
        plan.score_only(0, raw, self.dark, self.coeff, self.gains)
        # u32 order key -> int64 (MAX all-reduce on a signed type keeps the order)
        return plan.scores[0], plan.max_key[0:1].view(torch.int32).to(torch.int64) & 0xFFFFFFFF

    def topk_init(self, n_total: int, k: int):
        _lib.call("skyrx_topk_init", n_total, k, self.plan.topk_ws.data_ptr(), _dev.stream_ptr())

    def topk_hist(self, scores, digit: int) -> torch.Tensor:
        _lib.call("skyrx_topk_hist", scores.data_ptr(), scores.numel(), digit,
                  self.plan.topk_ws.data_ptr(), _dev.stream_ptr())
        return self.plan.topk_hist_view()

    def topk_pick(self, digit: int):
        _lib.call("skyrx_topk_pick", digit, self.plan.topk_ws.data_ptr(),
                  self.plan.thr[0:1].data_ptr(), _dev.stream_ptr())

    def threshold(self) -> float:
        return float(self.plan.thr[0].item())

    def mask(self, scores):
        _lib.call("skyrx_mask_gt", scores.data_ptr(), scores.numel(),
                  self.plan.thr[0:1].data_ptr(), self.plan.mask[0].data_ptr(), _dev.stream_ptr())
        return self.plan.mask[0].view(torch.bool)

    key_to_float = staticmethod(key_to_float)


def global_detect(raw_block, ops, n_total: int, group=None, k: int | None = None):
    """Run the R-GLOBAL protocol on this rank's block (collectives on `group`)."""
    # every collective runs whenever a process group exists (N = 1 included, so
    # the NCCL path is exercised on a single-GPU lease); none without one
    distributed = dist.is_available() and dist.is_initialized()

    def allreduce(t, op):
        if distributed:
            dist.all_reduce(t, op=op, group=group)
        return t

    # 1. common shift from the first block
    shift = ops.shift(raw_block)
    if distributed:
        dist.broadcast(shift, src=dist.get_global_rank(group, 0) if group is not None else 0,
                       group=group)
    # 2. moments + flags, summed / or-ed over ranks; identical finalize everywhere
    moments, nonfinite = ops.moments(raw_block, shift)
    allreduce(moments, dist.ReduceOp.SUM)
    allreduce(nonfinite, dist.ReduceOp.MAX)
    stats = ops.finalize(moments, shift, nonfinite)
    host_stats = ops.check(stats, n_total)
    # 3. scores of this block and the global max
    scores, maxkey = ops.score(raw_block)
    allreduce(maxkey, dist.ReduceOp.MAX)
    # 4. global top-k threshold by histogram all-reduce, then the local mask
    k = topk_count(n_total) if k is None else int(k)
    ops.topk_init(n_total, k)
    for digit in range(3):
        allreduce(ops.topk_hist(scores, digit), dist.ReduceOp.SUM)
        ops.topk_pick(digit)
    mask = ops.mask(scores)
    return GlobalDetection(host_stats, scores, mask, ops.threshold(),
                           ops.key_to_float(maxkey[0]), n_total)


class GlobalRX:
    """Convenience wrapper: one rank's block of a line-partitioned mosaic."""

    def __init__(self, lines_local: int, samples: int, bands: int, tables, n_total: int,
                 group=None):
        self.ops = CudaOps(lines_local, samples, bands, tables)
        self.n_total = n_total
        self.group = group

    def detect(self, raw_block, gains=None, k: int | None = None) -> GlobalDetection:
        self.ops.set_gains(gains)
        raw = raw_block if isinstance(raw_block, torch.Tensor) else _dev.to_device(
            np.asarray(raw_block), torch.uint16)
        return global_detect(raw, self.ops, self.n_total, self.group, k)
