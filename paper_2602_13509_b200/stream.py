"""R-STREAM: line-by-line detection with an exponentially forgetting background.

BASELINE config 2 (SURVEY.md §8(a) R-STREAM): 249-line chunks of the 900 x 70
geometry (1 s at the paper's line rate), background updated
per chunk with forgetting factor 0.99 and Sigma^-1 recomputed per chunk.  The
reference has no streaming detector; the frozen definition (and its CPU
restatement, oracle/skyrx_oracle.py StreamingStats) is:

    state (n, s, Q) in f64 about a fixed shift c (set from chunk 0)
    per chunk:  n <- lam n + m,  s <- lam s + sum(x - c),  Q <- lam Q + sum((x-c)(x-c)^T)
    mu = c + s/n,  Sigma = (Q - s s^T / n) / (n - 1)  -> rx.py:68-86 factorisation
    score the chunk with the stats that already include it; mask = top 0.1 %.

Chunk 0 therefore reduces to compute_stats/rx_scores on chunk 0, which the
reference pins.  Everything per chunk stays on the device: K2 moments of the
chunk (f64, the chunk is small), the fold (skyrx_moments_fold), K3 finalize,
K4 score and the top-k select.  From chunk 1 on the fixed chain is replayed
from one CUDA graph, so a chunk costs one graph launch plus its copies.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .calibrate import line_gains, tables_of
from .rx import CubeStats, DetectPlan, constant_gain, key_to_float, topk_count


@dataclass
class ChunkResult:
    """Scores / mask of one chunk and the background they were scored against."""

    index: int
    scores: object       # (lines, samples) f32 (numpy for host input, tensor for device input)
    mask: object         # (lines, samples) bool, top 0.1 % of the chunk
    threshold: float     # delta_(k+1) of the chunk
    max_score: float
    stats: CubeStats | None = None   # host copy, only when update(..., with_stats=True)


class StreamingRX:
    """Per-chunk RX detector with an exponentially forgetting background.

    ``update(raw_chunk)`` takes a RawCube-like object (``values`` u16 (L, S, B),
    optional line gains) or a bare u16 array / CUDA tensor of one chunk and
    returns its :class:`ChunkResult`.  Chunks must all have ``chunk_lines``
    lines (the geometry of the captured graph).
    """

    def __init__(self, tables, chunk_lines: int = 249, forget: float = 0.99,
                 k: int | None = None, use_graph: bool = True):
        self.tables = tables_of(tables)
        S, B = self.tables.samples, self.tables.bands
        if not 0.0 < forget <= 1.0:
            raise ValueError(f"forget factor {forget} outside (0, 1]")
        self.shape = (chunk_lines, S, B)
        self.forget = float(forget)
        self.k = topk_count(chunk_lines * S) if k is None else int(k)
        self.plan = DetectPlan(chunk_lines, S, B)
        self.dark, self.coeff = self.tables.device()
        self.raw = _dev.zeros(self.shape, torch.int16).view(torch.uint16)
        self.gains = _dev.zeros((chunk_lines,), torch.float32) + 1.0
        nm = int(_lib.load().skyrx_moments_len(B))
        self.chunk_moments = _dev.zeros((nm,), torch.float64)
        self.prev_state = _dev.zeros((nm,), torch.float64)
        lib = _lib.load()
        # exact raw-byte moments on the tensor cores when the chunk geometry allows
        self.raw_ok = bool(lib.skyrx_stats_raw_supported(chunk_lines, S, B, self.raw.data_ptr()))
        self.use_graph = use_graph
        self.graph = None
        self.chunks = 0
        self.gain = 1.0

    # ------------------------------------------------------------------ device chain
    def _enqueue(self, first: bool, gain: float | None, precise: bool = False):
        """The per-chunk device chain.  gain = the chunk's common line gain (None if
        the lines differ): then, unless ``precise``, the moments are the exact
        raw-byte tensor-core Grams; otherwise the f64 kernel."""
        L, S, B = self.shape
        plan, ds = self.plan, self.plan.ds
        s = _dev.stream_ptr()
        args = (self.raw.data_ptr(), L, S, B, self.dark.data_ptr(), self.coeff.data_ptr(),
                self.gains.data_ptr())
        ds.flags.zero_()
        if first:
            _lib.call("skyrx_stats_shift", _lib.IN_RAW_U16, *args, ds.shift[0].data_ptr(), s)
        use_raw = self.raw_ok and gain is not None and not precise
        plan.used_raw[0] = use_raw
        plan.gain_one[0] = gain == 1.0
        plan.gain_val[0] = gain
        if use_raw:
            _lib.call("skyrx_stats_raw", self.raw.data_ptr(), L, S, B, self.dark.data_ptr(),
                      self.coeff.data_ptr(), float(gain), ds.shift[0].data_ptr(),
                      self.chunk_moments.data_ptr(), ds.flags.data_ptr(), plan.raw_ws.data_ptr(),
                      plan.raw_ws_bytes, s)
        else:
            _lib.call("skyrx_stats_accumulate", _lib.IN_RAW_U16, *args, ds.shift[0].data_ptr(),
                      1, self.chunk_moments.data_ptr(), ds.flags.data_ptr(), plan.ws.data_ptr(),
                      plan.ws_bytes, s)
        # fold, keeping the pre-chunk state as the undo point if this chunk must be redone
        _lib.call("skyrx_moments_fold_keep", ds.moments[0].data_ptr(),
                  self.chunk_moments.data_ptr(), B, self.forget, self.prev_state.data_ptr(), s)
        plan.finalize()
        plan.score(0, self.raw, self.dark, self.coeff, self.gains, self.k)

    def _run(self, gain):
        if self.chunks == 0:
            self.plan.ds.moments.zero_()
            self._enqueue(first=True, gain=gain)
            return
        if not self.use_graph or gain != 1.0:
            self._enqueue(first=False, gain=gain)
            return
        if self.graph is None:
            # capture the steady-state chain once (shift fixed, buffers static, gain 1)
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                self._enqueue(first=False, gain=1.0)
            torch.cuda.current_stream().wait_stream(side)
            self.graph = g
        self.graph.replay()
        self.plan.used_raw[0] = self.raw_ok
        self.plan.gain_one[0] = True
        self.plan.gain_val[0] = 1.0

    # ------------------------------------------------------------------ public API
    def update(self, chunk, *, with_stats: bool = False) -> ChunkResult:
        values = chunk if isinstance(chunk, (torch.Tensor, np.ndarray)) else chunk.values
        L, S, B = self.shape
        if tuple(values.shape) != self.shape:
            raise ValueError(f"chunk shape {tuple(values.shape)} != stream geometry {self.shape}")
        on_dev = _dev.is_device(values)
        if isinstance(values, torch.Tensor):
            self.raw.copy_(values.view(torch.uint16) if values.dtype != torch.uint16 else values,
                           non_blocking=True)
        else:
            a = np.ascontiguousarray(np.asarray(values, np.uint16))
            self.raw.copy_(torch.from_numpy(a.view(np.int16)).view(torch.uint16),
                           non_blocking=True)
        gain = 1.0
        if getattr(chunk, "gains", None) is not None or len(getattr(chunk, "line_meta", ())):
            g = line_gains(chunk)
            gain = constant_gain(g, self.tables)
            g = g if isinstance(g, torch.Tensor) else torch.from_numpy(np.asarray(g, np.float32))
            self.gains.copy_(g, non_blocking=True)
        else:
            self.gains.fill_(1.0)
        first = self.chunks == 0
        self._run(gain)
        ds = self.plan.ds
        if int(ds.status[0].item()) == _lib.ERR_RANGE:
            # a value below dark (clamp): the raw-byte moments do not apply -> redo
            # this chunk's moments in f64 from the pre-chunk state
            ds.moments[0].copy_(self.prev_state)
            if first:
                ds.moments[0].zero_()
            self._enqueue(first=first, gain=gain, precise=True)
        ds.check(0, L * S)  # synchronises: raises the reference's errors
        idx = self.chunks
        self.chunks += 1
        thr = float(self.plan.thr[0].item())
        mx = key_to_float(self.plan.max_key[0])
        stats = ds.host(0, L * S) if with_stats else None
        if on_dev:
            return ChunkResult(idx, self.plan.scores[0].clone(),
                               self.plan.mask[0].to(torch.bool), thr, mx, stats)
        return ChunkResult(idx, _dev.to_host(self.plan.scores[0]),
                           _dev.to_host(self.plan.mask[0]).view(bool), thr, mx, stats)

    def reset(self):
        """Forget the background (the next chunk re-seeds the shift).  The captured
        chunk graph stays valid: it reads the shift and state from device buffers."""
        self.chunks = 0
