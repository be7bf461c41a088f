"""Global RX detector on the B200 — drop-in for skyrx.rx.

Reference: rx.py:26-124.  Public names, signatures, return types and error
messages are the reference's; the work runs in CUDA kernels:

    compute_stats   K2 moments (csrc/stats.cu gram_kernel) + K3 factorisation
    rx_scores       K4 whitening product (csrc/score.cu)
    normalize/threshold/transmit_domain/top-k   K5 (csrc/select.cu)

Two arithmetic modes, both parity-tested:
  * ``"precise"`` (default for the drop-in functions): FP64 products and
    sums everywhere, so the reference's own suites pass at their tolerances
    (1e-9 permutation / backend agreement, 1e-6 oracles).
  * ``"fast"`` (``detect()``, bench.py): FP32 Gram blocks of <= 192 products
    promoted to FP64, FP32 whitening — within BASELINE's 1e-5 (stats) and 1e-4
    (scores) and several times faster.

``detect()`` is the fused hot path the pipeline's calibrate+detect stages need
(pipeline.py:167-175): raw -> moments -> factor -> scores -> top-0.1% mask
without materialising radiance, device-resident end to end, one host sync.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev, _lib
from .calibrate import _check_tables, _out_cls, _raw_device, line_gains, tables_of
from .cube import ScoreMap

RIDGE_EPSILONS = (1e-10, 1e-9, 1e-8, 1e-7, 1e-6)
MODES = ("precise", "fast")
TC_MIN_PIXELS = 1 << 18   # below this detect() fits the background in f64

_STATUS_MSG = {
    _lib.ERR_NONFINITE: "invalid data: cube contains non-finite values",
    _lib.ERR_NOT_PD: "covariance not positive definite even after ridging",
}


@dataclass(frozen=True)
class CubeStats:
    """rx.py:26-39: band means, covariance, its inverse, ridge and Cholesky factor."""

    mu: np.ndarray
    sigma: np.ndarray
    sigma_inv: np.ndarray
    ridge_used: float
    chol_lower: np.ndarray
    _device: object = field(default=None, compare=False, repr=False)


def _bp(bands: int) -> int:
    return ((bands + 7) // 8) * 8


class DeviceStats:
    """Device-resident fit of one or more backgrounds (batched over strips).

    Arrays are (batch, ...) CUDA tensors; nothing is copied to the host until
    :meth:`host` (which also raises the reference's ValueErrors).
    """

    def __init__(self, bands: int, batch: int = 1):
        self.bands = bands
        self.batch = batch
        self.ld = _bp(bands)
        f64, f32 = torch.float64, torch.float32
        B = bands
        self.shift = _dev.zeros((batch, B), f64)
        self.moments = _dev.zeros((batch, int(_lib.load().skyrx_moments_len(B))), f64)
        self.flags = _dev.zeros((batch,), torch.int32)
        self.mu = _dev.empty((batch, B), f64)
        self.sigma = _dev.empty((batch, B, B), f64)
        self.chol = _dev.zeros((batch, B, B), f64)
        self.sigma_inv = _dev.empty((batch, B, B), f64)
        self.w64 = _dev.empty((batch, B, B), f64)
        self.whiten = _dev.zeros((batch, self.ld, self.ld), f32)
        self.mu_hilo = _dev.zeros((batch, 2 * B), f32)
        self.ridge = _dev.zeros((batch,), f64)
        self.status = _dev.zeros((batch,), torch.int32)

    def finalize(self, slot: int | None = None):
        """Factor every slot's moments, or only ``slot``."""
        sl = slice(None) if slot is None else slice(slot, slot + 1)
        n = self.batch if slot is None else 1
        t = lambda x: x[sl].data_ptr()  # noqa: E731
        _lib.call("skyrx_stats_finalize", t(self.moments), t(self.shift), t(self.flags),
                  self.bands, n, t(self.mu), t(self.sigma), t(self.chol), t(self.sigma_inv),
                  t(self.w64), t(self.whiten), self.ld, t(self.mu_hilo), t(self.ridge),
                  t(self.status), _dev.stream_ptr())
        return self

    def check(self, i: int = 0, npix: int | None = None):
        st = int(self.status[i].item())
        if st == _lib.ERR_INSUFFICIENT:
            n = npix if npix is not None else int(self.moments[i, 0].item())
            raise ValueError(f"insufficient samples: {n} pixels for {self.bands} bands")
        if st != _lib.OK:
            raise ValueError(_STATUS_MSG.get(st, f"stats failed with status {st}"))

    def host(self, i: int = 0, npix: int | None = None) -> CubeStats:
        self.check(i, npix)
        h = lambda t: _dev.to_host(t[i])  # noqa: E731
        return CubeStats(mu=h(self.mu), sigma=h(self.sigma), sigma_inv=h(self.sigma_inv),
                         ridge_used=float(self.ridge[i].item()), chol_lower=h(self.chol),
                         _device=(self, i))


def _radiance_device(cube) -> torch.Tensor:
    return _dev.to_device(cube.values, torch.float32)


def accumulate_moments(ds: DeviceStats, i: int, kind: int, pixels: torch.Tensor, lines: int,
                       samples: int, tables=None, gains=None, *, precise: bool,
                       shift: bool = True) -> None:
    """K2 for one cube into slot i of ``ds`` (shift, moments, non-finite flag)."""
    B = ds.bands
    dark = coeff = None
    if kind == _lib.IN_RAW_U16:
        dark, coeff = tables
    args = (pixels.data_ptr(), lines, samples, B, _dev.ptr(dark), _dev.ptr(coeff),
            _dev.ptr(gains))
    s = _dev.stream_ptr()
    if shift:
        _lib.call("skyrx_stats_shift", kind, *args, ds.shift[i].data_ptr(), s)
    nbytes = _lib.C.c_size_t(0)
    _lib.call("skyrx_stats_workspace", lines, samples, B, _lib.C.byref(nbytes))
    ws = _dev.empty((max(int(nbytes.value), 8),), torch.uint8)
    _lib.call("skyrx_stats_accumulate", kind, *args, ds.shift[i].data_ptr(), int(precise),
              ds.moments[i].data_ptr(), ds.flags[i:i + 1].data_ptr(), ws.data_ptr(),
              int(nbytes.value), s)


def compute_stats(cube, chunk: int = 65536, *, mode: str = "precise") -> CubeStats:
    """rx.py:42-86: per-cube Gaussian fit (mean, unbiased covariance, inverse).

    ``chunk`` is accepted for signature compatibility (results are
    chunk-invariant, rx.py's own test_chunked_equals_unchunked)."""
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}")
    bands = cube.bands
    n = cube.lines * cube.samples
    if n <= bands:
        raise ValueError(f"insufficient samples: {n} pixels for {bands} bands")
    ds = DeviceStats(bands)
    px = _radiance_device(cube)
    L, S = cube.lines, cube.samples
    if mode == "fast" and _tc_f32_moments(ds, px, L, S):
        ds.finalize()
        if int(ds.status[0].item()) != _lib.ERR_RANGE:
            return ds.host(0, n)
        ds.flags.zero_()  # the quantiser's range overflowed: the f32-run kernel below
    accumulate_moments(ds, 0, _lib.IN_F32, px, L, S, precise=(mode == "precise"))
    ds.finalize()
    return ds.host(0, n)


def _tc_f32_moments(ds: DeviceStats, px: torch.Tensor, L: int, S: int) -> bool:
    """mode="fast" moments of an f32 radiance cube on the tensor cores (skyrx_stats_tc_f32:
    quantised int8 digits, exact int32 digit Gram); False where the kernel does not apply
    (B > 79, small cubes whose quantiser noise does not average out, unaligned rows)."""
    B = ds.bands
    lib = _lib.load()
    if (B > 79 or L * S < TC_MIN_PIXELS or (S * B * 4) % 16 != 0
            or not lib.skyrx_stats_tc_supported(L, S, B, px.data_ptr())):
        return False
    s = _dev.stream_ptr()
    qinv = _dev.empty((B,), torch.float32)
    nbytes = int(lib.skyrx_stats_tc_workspace(B))
    ws = _dev.empty((nbytes,), torch.uint8)
    _lib.call("skyrx_quant_shift", _lib.IN_F32, px.data_ptr(), L, S, B, None, None, None,
              ds.shift[0].data_ptr(), qinv.data_ptr(), s)
    _lib.call("skyrx_stats_tc_f32", px.data_ptr(), L, S, B, ds.shift[0].data_ptr(),
              qinv.data_ptr(), ds.moments[0].data_ptr(), ds.flags[0:1].data_ptr(),
              ws.data_ptr(), nbytes, s)
    return True


def _device_whitening(stats: CubeStats, bands: int):
    d = stats._device
    if d is not None:
        ds, i = d
        return ds.whiten[i], ds.mu_hilo[i], ds.ld
    ld = _bp(bands)
    chol = _dev.to_device(np.asarray(stats.chol_lower, np.float64))
    mu = _dev.to_device(np.asarray(stats.mu, np.float64))
    w64 = _dev.empty((bands, bands), torch.float64)
    wf = _dev.zeros((ld, ld), torch.float32)
    mhl = _dev.empty((2 * bands,), torch.float32)
    _lib.call("skyrx_whiten_prepare", chol.data_ptr(), mu.data_ptr(), bands, w64.data_ptr(),
              wf.data_ptr(), ld, mhl.data_ptr(), _dev.stream_ptr())
    return wf, mhl, ld


def mahalanobis_sq_device(pixels: torch.Tensor, mu, chol) -> torch.Tensor:
    """_accel.py:75-90 semantics on device: f64 delta per row of (N, B) pixels."""
    n, b = pixels.shape
    kind = _lib.IN_F64 if pixels.dtype == torch.float64 else _lib.IN_F32
    if kind == _lib.IN_F32 and pixels.dtype != torch.float32:
        pixels = pixels.to(torch.float32)
    mu_d = _dev.to_device(mu, torch.float64)
    ch_d = _dev.to_device(chol, torch.float64)
    bp = _bp(b)
    ws = _dev.empty((b * b + bp * bp,), torch.float64)
    out = _dev.empty((n,), torch.float64)
    _lib.call("skyrx_mahalanobis_sq", kind, pixels.data_ptr(), n, b, mu_d.data_ptr(),
              ch_d.data_ptr(), ws.data_ptr(), out.data_ptr(), _dev.stream_ptr())
    return out


def rx_scores(cube, stats: CubeStats, *, mode: str = "precise") -> ScoreMap:
    """rx.py:89-97: squared Mahalanobis distance of every pixel, f32 (lines, samples)."""
    if stats.mu.shape[0] != cube.bands:
        raise ValueError(
            f"stats fitted for {stats.mu.shape[0]} bands, cube has {cube.bands}"
        )
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}")
    L, S, B = cube.lines, cube.samples, cube.bands
    px = _radiance_device(cube)
    if mode == "precise":
        d = mahalanobis_sq_device(px.reshape(-1, B), stats.mu, stats.chol_lower)
        out = d.to(torch.float32).reshape(L, S)
    else:
        wf, mhl, ld = _device_whitening(stats, B)
        out = _dev.empty((L, S), torch.float32)
        _lib.call("skyrx_score", _lib.IN_F32, px.data_ptr(), L, S, B, None, None, None,
                  mhl.data_ptr(), wf.data_ptr(), ld, out.data_ptr(), None, _dev.stream_ptr())
    cls = _out_cls(cube, "ScoreMap", ScoreMap)
    return cls(_dev.like_input(cube.values, out))


def _scores_device(scores) -> torch.Tensor:
    v = scores.values if hasattr(scores, "values") else scores
    return _dev.to_device(v, torch.float32)


def score_max_key(v: torch.Tensor) -> torch.Tensor:
    key = _dev.zeros((1,), torch.uint32)
    _lib.call("skyrx_max", v.data_ptr(), v.numel(), key.data_ptr(), _dev.stream_ptr())
    return key


def key_to_float(key: torch.Tensor) -> float:
    u = int(key.item())
    b = (u & 0x7FFFFFFF) if (u & 0x80000000) else (~u & 0xFFFFFFFF)
    return float(np.array([b], np.uint32).view(np.float32)[0])


def normalize_scores(scores) -> ScoreMap:
    """rx.py:100-105: divide by f32(max); an all-zero (max <= 0) map is returned as is."""
    v = _scores_device(scores)
    if v.numel() == 0:
        return scores
    key = score_max_key(v)
    out = _dev.empty(tuple(v.shape), torch.float32)
    _lib.call("skyrx_normalize", v.data_ptr(), v.numel(), key.data_ptr(), out.data_ptr(),
              _dev.stream_ptr())
    if key_to_float(key) <= 0.0:
        return scores
    cls = _out_cls(scores, "ScoreMap", ScoreMap)
    return cls(_dev.like_input(scores.values, out))


def threshold_scores(norm_scores, threshold: float):
    """rx.py:108-112: mask = values > threshold, compared in f32 (NEP 50)."""
    if not 0.0 <= threshold <= 1.0:
        raise ValueError(f"threshold {threshold} outside [0, 1]")
    v = _scores_device(norm_scores)
    mask = _dev.empty(tuple(v.shape), torch.uint8)
    _lib.call("skyrx_threshold", v.data_ptr(), v.numel(), float(np.float32(threshold)),
              mask.data_ptr(), _dev.stream_ptr())
    return _dev.like_input(norm_scores.values, mask.to(torch.bool))


def transmit_domain(values, max_score: float):
    """rx.py:115-124: sqrt(score / cube max) in f64; zeros when the max is 0."""
    v = _dev.to_device(values, torch.float32)
    out = _dev.empty(tuple(v.shape), torch.float64)
    _lib.call("skyrx_transmit_domain", v.data_ptr(), v.numel(), float(max_score),
              out.data_ptr(), _dev.stream_ptr())
    return _dev.like_input(values, out)


# --------------------------------------------------------------------------- R-TOPK
def topk_cand_cap(n: int) -> int:
    """Candidate slots of skyrx_topk_mask: the top-11-bit bin holding the
    threshold rarely holds more than a few k values; beyond this the kernel
    rescans (exact, slower)."""
    return n // 64 + 4096


def topk_count(n: int) -> int:
    """k = ceil(0.001 * N) in integers (SURVEY.md §8(a) R-TOPK)."""
    return (n + 999) // 1000


def topk_threshold_device(v: torch.Tensor, k: int) -> torch.Tensor:
    ws = _dev.empty((int(_lib.load().skyrx_topk_workspace()) // 4 + 4,), torch.int32)
    thr = _dev.empty((1,), torch.float32)
    _lib.call("skyrx_topk_threshold", v.data_ptr(), v.numel(), k, thr.data_ptr(),
              ws.data_ptr(), _dev.stream_ptr())
    return thr


def topk_mask_device(v: torch.Tensor, k: int, cand_cap: int | None = None):
    """(mask u8, thr) of R-TOPK on device scores in one mask pass
    (skyrx_topk_mask); ``cand_cap`` overrides the candidate slots (tests)."""
    n = v.numel()
    cap = topk_cand_cap(n) if cand_cap is None else int(cand_cap)
    ws = _dev.empty((int(_lib.load().skyrx_topk_workspace()) // 4 + 4,), torch.int32)
    cand = _dev.empty((2 * max(cap, 1),), torch.int32)
    thr = _dev.empty((1,), torch.float32)
    mask = _dev.empty(tuple(v.shape), torch.uint8)
    s = _dev.stream_ptr()
    _lib.call("skyrx_topk_init", n, k, ws.data_ptr(), s)
    _lib.call("skyrx_topk_mask", v.data_ptr(), n, 0, thr.data_ptr(), mask.data_ptr(),
              ws.data_ptr(), cand.data_ptr(), cap, s)
    return mask, thr


def topk_mask(scores, k: int | None = None):
    """R-TOPK: mask = delta > delta_(k+1), the top ceil(0.1%) of raw f32 scores."""
    v = _scores_device(scores).contiguous()
    k = topk_count(v.numel()) if k is None else int(k)
    mask, _ = topk_mask_device(v, k)
    src = scores.values if hasattr(scores, "values") else scores
    return _dev.like_input(src, mask.to(torch.bool))


# --------------------------------------------------------------------------- fused hot path
@dataclass
class Detection:
    """Result of :func:`detect`: host numpy or device tensors (``device=True``)."""

    stats: object       # CubeStats (host) or DeviceStats (device)
    scores: object      # (L, S) f32
    mask: object        # (L, S) bool (top 0.1%)
    threshold: float    # delta_(k+1)
    max_score: float


class DetectPlan:
    """Reusable device buffers for repeated detect() calls on one cube shape."""

    def __init__(self, lines: int, samples: int, bands: int, batch: int = 1):
        self.shape = (lines, samples, bands)
        self.ds = DeviceStats(bands, batch)
        nbytes = _lib.C.c_size_t(0)
        _lib.call("skyrx_stats_workspace", lines, samples, bands, _lib.C.byref(nbytes))
        self.ws_bytes = int(nbytes.value)
        self.ws = _dev.empty((max(self.ws_bytes, 8),), torch.uint8)
        self.scores = _dev.empty((batch, lines, samples), torch.float32)
        self.mask = _dev.empty((batch, lines, samples), torch.uint8)
        self.max_key = _dev.zeros((batch,), torch.uint32)
        self.thr = _dev.empty((batch,), torch.float32)
        self.topk_ws = _dev.empty((int(_lib.load().skyrx_topk_workspace()) // 4 + 4,),
                                  torch.int32)
        # (index, key) slots for the scores inside the threshold's top digit bin
        self.cand_cap = topk_cand_cap(lines * samples)
        self.cand = _dev.empty((2 * self.cand_cap,), torch.int32)
        self.launches = 0
        # per slot: every line gain is exactly 1 (set by run(); lets the score
        # kernel drop the per-line gain from its transform)
        self.gain_one = [False] * batch
        self.gain_val = [None] * batch
        self.used_raw = [False] * batch   # raw-byte moments ran (no-clamp proof available)
        lib = _lib.load()
        use_tc = os.environ.get("SKYRX_B200_TC", "1") != "0"
        self.tc = bands <= 80 and use_tc              # tensor-core score kernel
        self.tc_stats = bands <= 79 and use_tc        # tensor-core moments kernel
        self.wpack_bytes = int(lib.skyrx_wpack_bytes(bands)) if self.tc else 0
        self.wpack = (_dev.empty((batch, self.wpack_bytes), torch.uint8) if self.tc else None)
        self.qinv = _dev.zeros((batch, bands), torch.float32)
        self.tc_ws_bytes = int(lib.skyrx_stats_tc_workspace(bands)) if self.tc_stats else 0
        self.tc_ws = _dev.empty((max(self.tc_ws_bytes, 8),), torch.uint8)
        self.raw_stats = bands <= 272 and use_tc and os.environ.get("SKYRX_B200_RAWGRAM", "1") != "0"
        # (with room for the clamp correction's pixel bitmap, skyrx_stats_raw_workspace_for)
        self.raw_ws_bytes = (int(lib.skyrx_stats_raw_workspace_for(lines, samples, bands))
                             if self.raw_stats else 0)
        self.raw_ws = _dev.empty((max(self.raw_ws_bytes, 8),), torch.uint8)
        # exact-digit score kernel (per-sample records, B <= 128): the path for
        # 80 < B <= 128 (K4-TC's tables no longer fit); SKYRX_B200_TCS=1 forces it
        # for smaller B too, =0 disables it
        tcs_env = os.environ.get("SKYRX_B200_TCS", "")
        self.tcs = self.raw_stats and tcs_env != "0" and (bands > 80 or tcs_env == "1")
        self.rec_bytes = int(lib.skyrx_score_rec_bytes(bands)) * samples if self.tcs else 0
        # ... and its wide form for 128 < B <= 272 (N-blocked V_s), whatever moments path
        self.tcw = 128 < bands <= 272 and use_tc and tcs_env != "0"
        if self.tcw:
            self.rec_bytes = int(lib.skyrx_scorew_rec_bytes(bands)) * samples
        self.records = (_dev.empty((batch, self.rec_bytes), torch.uint8)
                        if (self.tcs or self.tcw) else None)

    def run(self, i: int, raw: torch.Tensor, dark, coeff, gains, k: int | None = None,
            precise: bool = False, force_ffma: bool = False, gain_const: float | None = None,
            events=None):
        """Enqueue the moments of cube i (no host synchronisation).  ``events`` =
        (start, end) CUDA events recorded around the moments kernel call alone."""
        return self._moments(i, raw, dark, coeff, gains, precise, force_ffma, gain_const, True,
                             events)

    def run_moments(self, i: int, raw: torch.Tensor, dark, coeff, gains, precise: bool = False,
                    force_ffma: bool = False, gain_const: float | None = None):
        """Moments of cube i about the shift already in ``ds.shift[i]`` (R-GLOBAL:
        a shift common to every rank's block)."""
        return self._moments(i, raw, dark, coeff, gains, precise, force_ffma, gain_const, False)

    def _moments(self, i, raw, dark, coeff, gains, precise, force_ffma, gain_const, own_shift,
                 events=None):
        L, S, B = self.shape
        ds = self.ds
        s = _dev.stream_ptr()
        args = (raw.data_ptr(), L, S, B, dark.data_ptr(), coeff.data_ptr(), gains.data_ptr())
        self.gain_one[i] = gain_const == 1.0
        self.gain_val[i] = gain_const
        self.used_raw[i] = False
        ds.flags[i].zero_()
        lib = _lib.load()
        # the raw-byte path is exact at any size; small cubes skip only the int8
        # quantiser (its noise averages out over many pixels); a quantiser overflow
        # or a clamp is redone in f64 (force_ffma)
        small = L * S < TC_MIN_PIXELS
        precise = precise or force_ffma
        if (self.raw_stats and not precise and gain_const is not None
                and lib.skyrx_stats_raw_supported(L, S, B, raw.data_ptr())):
            # exact integer byte Grams on the tensor cores (constant line gain); with
            # its own shift the call centres on f32(mean) itself (no shift pass)
            self.used_raw[i] = True
            if events is not None:
                events[0].record()
            _lib.call("skyrx_stats_raw_own_shift" if own_shift else "skyrx_stats_raw",
                      raw.data_ptr(), L, S, B, dark.data_ptr(),
                      coeff.data_ptr(), float(gain_const), ds.shift[i].data_ptr(),
                      ds.moments[i].data_ptr(), ds.flags[i:i + 1].data_ptr(),
                      self.raw_ws.data_ptr(), self.raw_ws_bytes, s)
            if events is not None:
                events[1].record()
        elif (self.tc_stats and not precise and not small and own_shift
                and lib.skyrx_stats_tc_supported(L, S, B, raw.data_ptr())):
            _lib.call("skyrx_quant_shift", _lib.IN_RAW_U16, *args, ds.shift[i].data_ptr(),
                      self.qinv[i].data_ptr(), s)
            _lib.call("skyrx_stats_tc", *args, ds.shift[i].data_ptr(), self.qinv[i].data_ptr(),
                      ds.moments[i].data_ptr(), ds.flags[i:i + 1].data_ptr(),
                      self.tc_ws.data_ptr(), self.tc_ws_bytes, s)
        else:
            # the general kernel in f64 products (precise): its f32-product mode moves
            # Sigma by ~5e-8, which cond(Sigma) ~1e4 turns into > 1e-5 on Sigma^-1
            if own_shift:
                _lib.call("skyrx_stats_shift", _lib.IN_RAW_U16, *args, ds.shift[i].data_ptr(), s)
            _lib.call("skyrx_stats_accumulate", _lib.IN_RAW_U16, *args, ds.shift[i].data_ptr(),
                      1, ds.moments[i].data_ptr(), ds.flags[i:i + 1].data_ptr(),
                      self.ws.data_ptr(), self.ws_bytes, s)
        self.launches += 3
        return self

    def recover_range(self, cubes) -> list[int]:
        """Redo (synchronously) any cube whose tensor-core quantiser overflowed.

        ``cubes[i] = (raw, dark, coeff, gains)``.  Returns the recomputed slots."""
        st = self.ds.status.cpu().numpy()
        redo = [i for i in cubes if st[i] == _lib.ERR_RANGE]
        if redo:
            for i in redo:
                self.run(i, *cubes[i], force_ffma=True)
            self.finalize()
            for i in redo:
                self.score(i, *cubes[i])
        # the exact-digit score kernels could not apply (raw counts >= 4096: 16, or no
        # no-clamp proof: 32): rescore with the general kernels
        fl = self.ds.flags.cpu().numpy()
        rescore = [i for i in cubes if fl[i] & 48]
        for i in rescore:
            self.used_raw[i] = False
            keep, self.tcw = self.tcw, False
            self.score(i, *cubes[i])
            self.tcw = keep
        return sorted(set(redo) | set(rescore))

    def finalize(self, slot: int | None = None):
        self.ds.finalize(slot)
        self.launches += 1
        if self.tc:
            sl = slice(None) if slot is None else slice(slot, slot + 1)
            _lib.call("skyrx_pack_whiten", self.ds.w64[sl].data_ptr(), self.ds.bands,
                      self.ds.batch if slot is None else 1, self.wpack[sl].data_ptr(),
                      _dev.stream_ptr())
            self.launches += 1
        return self

    def topk_hist_view(self) -> torch.Tensor:
        """The radix histogram inside the top-k workspace (int32 view, for all-reduce)."""
        off = 32 // 4
        return self.topk_ws[off:off + int(_lib.load().skyrx_topk_hist_len())]

    def score(self, i: int, raw: torch.Tensor, dark, coeff, gains, k: int | None = None,
              events=None):
        """Enqueue scores, top-k threshold and mask of cube i.  ``events`` =
        (start, end) CUDA events recorded around the score kernel alone."""
        L, S, B = self.shape
        n = L * S
        k = topk_count(n) if k is None else int(k)
        s = _dev.stream_ptr()
        ws = self.topk_ws.data_ptr()
        # R-TOPK as init -> (digit-0 histogram fused into the score kernel) ->
        # one mask pass (digit-0 pick per CTA, in-bin candidates appended) ->
        # digits 1 and 2 on the candidates
        _lib.call("skyrx_topk_init", n, k, ws, s)
        fused = self.score_only(i, raw, dark, coeff, gains, events, topk_hist0=True)
        sc = self.scores[i]
        thr = self.thr[i:i + 1].data_ptr()
        _lib.call("skyrx_topk_mask", sc.data_ptr(), n, int(fused), thr, self.mask[i].data_ptr(),
                  ws, self.cand.data_ptr(), self.cand_cap, s)
        self.launches += 1 + (2 if fused else 3)
        return self

    def score_only(self, i: int, raw: torch.Tensor, dark, coeff, gains, events=None,
                   topk_hist0: bool = False) -> bool:
        """Scores of cube i and their max key (no threshold / mask).  With
        ``topk_hist0`` the tensor-core kernel also adds the digit-0 top-k
        histogram into the top-k workspace; returns whether it did."""
        L, S, B = self.shape
        ds = self.ds
        s = _dev.stream_ptr()
        self.max_key[i].zero_()
        sc = self.scores[i]
        if events is not None:
            events[0].record()
        fused = False
        lib = _lib.load()
        hist = lib.skyrx_topk_histogram(self.topk_ws.data_ptr()) if topk_hist0 else None
        if (self.tcs and self.used_raw[i]
                and lib.skyrx_score_tcs_supported(L, S, B, raw.data_ptr())):
            # exact integer digits: needs the raw path's no-clamp proof (a clamp
            # makes the moments status ERR_RANGE and recover_range rescored generally)
            rec = self.records[i].data_ptr()
            _lib.call("skyrx_score_prep", ds.w64[i].data_ptr(), ds.mu_hilo[i].data_ptr(), S, B,
                      dark.data_ptr(), coeff.data_ptr(), float(self.gain_val[i]), 1, rec, s)
            _lib.call("skyrx_score_tcs", raw.data_ptr(), L, S, B, rec,
                      ds.flags[i:i + 1].data_ptr(), sc.data_ptr(),
                      self.max_key[i:i + 1].data_ptr(), hist, s)
            fused = topk_hist0
            self.launches += 1
        elif (self.tcw and self.gain_val[i] is not None
                and lib.skyrx_scorew_supported(L, S, B, raw.data_ptr())):
            # wide exact-digit kernel; it checks the no-clamp proof itself (flags |= 32
            # when missing: recover_range rescores generally)
            rec = self.records[i].data_ptr()
            _lib.call("skyrx_scorew_prep", ds.w64[i].data_ptr(), ds.mu_hilo[i].data_ptr(), S, B,
                      dark.data_ptr(), coeff.data_ptr(), float(self.gain_val[i]), 1, rec, s)
            _lib.call("skyrx_scorew", raw.data_ptr(), L, S, B, rec,
                      ds.flags[i:i + 1].data_ptr(), sc.data_ptr(),
                      self.max_key[i:i + 1].data_ptr(), hist, s)
            fused = topk_hist0
            self.launches += 1
        elif self.tc and lib.skyrx_score_tc_supported(L, S, B, raw.data_ptr()):
            _lib.call("skyrx_score_tc", raw.data_ptr(), L, S, B, dark.data_ptr(),
                      coeff.data_ptr(), None if self.gain_one[i] else gains.data_ptr(),
                      ds.mu_hilo[i].data_ptr(),
                      self.wpack[i].data_ptr(), ds.flags[i:i + 1].data_ptr(), sc.data_ptr(),
                      self.max_key[i:i + 1].data_ptr(), hist, s)
            fused = topk_hist0
        else:
            _lib.call("skyrx_score", _lib.IN_RAW_U16, raw.data_ptr(), L, S, B, dark.data_ptr(),
                      coeff.data_ptr(), gains.data_ptr(), ds.mu_hilo[i].data_ptr(),
                      ds.whiten[i].data_ptr(), ds.ld, sc.data_ptr(),
                      self.max_key[i:i + 1].data_ptr(), s)
        if events is not None:
            events[1].record()
        self.launches += 1
        return fused


def constant_gain(gains, tables) -> float | None:
    """The common line gain if every line shares it (and calibration cannot
    overflow f32), else None — the raw-byte moments path needs one gain."""
    g = gains.detach().cpu().numpy() if isinstance(gains, torch.Tensor) else np.asarray(gains)
    if g.size == 0 or not (g == g.flat[0]).all():
        return None
    g0 = float(np.float32(g.flat[0]))
    if not g0 > 0.0:
        return None
    # a non-finite dark entry makes radiance non-finite (rx.py:53-54); only the
    # general moments kernel flags that, so leave such tables to it
    if not np.isfinite(np.asarray(tables.dark, np.float32)).all():
        return None
    if not np.isfinite(np.float32(65535.0) * np.float32(tables.coeff.max()) / np.float32(g0)):
        return None
    return g0


def detect(raw, tables, *, k: int | None = None, device: bool | None = None,
           precise: bool = False, plan: DetectPlan | None = None) -> Detection:
    """Fused calibrate + RX + top-0.1% mask for one raw cube (the hot path).

    Equivalent to ``compute_stats(apply_calibration(raw))`` -> ``rx_scores`` ->
    ``topk_mask`` (oracle ``detect``), without materialising radiance.
    Raises the reference's ValueErrors (invalid tables, gains, insufficient,
    non-finite, not positive definite).
    """
    tables = tables_of(tables)
    _check_tables(raw, tables)
    gains = line_gains(raw)
    L, S, B = raw.lines, raw.samples, raw.bands
    n = L * S
    if n <= B:
        raise ValueError(f"insufficient samples: {n} pixels for {B} bands")
    dark, coeff = tables.device()
    rv = _raw_device(raw)
    gd = _dev.to_device(gains, torch.float32)
    plan = plan or DetectPlan(L, S, B)
    gain_const = constant_gain(gains, tables)
    plan.run(0, rv, dark, coeff, gd, precise=precise, gain_const=gain_const)
    plan.finalize().score(0, rv, dark, coeff, gd, k)
    plan.recover_range({0: (rv, dark, coeff, gd)})
    on_dev = _dev.is_device(raw.values) if device is None else device
    ds = plan.ds
    ds.check(0, n)
    thr = float(plan.thr[0].item())
    mx = key_to_float(plan.max_key[0])
    if on_dev:
        return Detection(ds, plan.scores[0], plan.mask[0].to(torch.bool), thr, mx)
    return Detection(ds.host(0, n), _dev.to_host(plan.scores[0]),
                     _dev.to_host(plan.mask[0]).view(bool), thr, mx)


def detect_batch(raws, tables, *, k: int | None = None,
                 plan: DetectPlan | None = None) -> list[Detection]:
    """:func:`detect` over a sequence of HOST cubes of one shape, pipelined.

    Two device slots: while the GPU works on cube i, the copy stream uploads cube
    i + 1 and downloads the scores, mask and statistics of cube i - 1 (PCIe is full
    duplex), so a stream of strips runs at the host-link rate.  ``tables`` is one
    CalibrationTables for all cubes or one per cube.  Results are host numpy
    (pinned) like :func:`detect`; a cube whose fast path did not apply (clamp,
    counts >= 4096) is redone with :func:`detect` after the pipeline drains.
    """
    raws = list(raws)
    if not raws:
        return []
    tabs = list(tables) if isinstance(tables, (list, tuple)) else [tables] * len(raws)
    if len(tabs) != len(raws):
        raise ValueError("one CalibrationTables per cube, or one for all")
    L, S, B = raws[0].lines, raws[0].samples, raws[0].bands
    for r in raws:
        if (r.lines, r.samples, r.bands) != (L, S, B):
            raise ValueError("detect_batch: every cube must have the same shape")
    n = L * S
    if n <= B:
        raise ValueError(f"insufficient samples: {n} pixels for {B} bands")
    plan = plan or DetectPlan(L, S, B, batch=2)
    if plan.ds.batch < 2 or plan.shape != (L, S, B):
        raise ValueError("detect_batch needs a DetectPlan of this shape with batch >= 2")
    dev = _dev.require_cuda()
    comp = torch.cuda.current_stream()
    copy = torch.cuda.Stream()
    bufs = [torch.empty((L, S, B), dtype=torch.uint16, device=dev) for _ in range(2)]
    nm = plan.ds.moments.shape[1]
    ev = lambda: torch.cuda.Event()  # noqa: E731
    h2d, comp_done, d2h = [], [], []
    outs = []
    for i, cube in enumerate(raws):
        j = i % 2
        tab = tables_of(tabs[i])
        _check_tables(cube, tab)
        gains = line_gains(cube)
        gain_const = constant_gain(gains, tab)
        dark, coeff = tab.device()
        v = cube.values
        src = v if isinstance(v, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(v))
        h2d.append(ev())
        with torch.cuda.stream(copy):
            if i >= 2:
                copy.wait_event(comp_done[i - 2])  # slot j's raw buffer is free
            bufs[j].copy_(src.view(torch.uint16) if src.dtype != torch.uint16 else src,
                          non_blocking=True)
            h2d[i].record(copy)
        comp.wait_event(h2d[i])
        if i >= 2:
            comp.wait_event(d2h[i - 2])  # slot j's outputs were downloaded
        # gains: a pinned staging copy, so the upload does not block the host (a pageable
        # copy would wait for the compute stream and serialise the pipeline)
        gsrc = gains if isinstance(gains, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(gains, np.float32))
        gd = gsrc.to(dev, non_blocking=True) if gsrc.is_cuda else \
            gsrc.pin_memory().to(dev, non_blocking=True)
        plan.run(j, bufs[j], dark, coeff, gd, gain_const=gain_const)
        plan.finalize(j).score(j, bufs[j], dark, coeff, gd, k)
        comp_done.append(ev())
        comp_done[i].record(comp)
        o = {name: torch.empty(shape, dtype=dt, pin_memory=True) for name, shape, dt in (
            ("scores", (L, S), torch.float32), ("mask", (L, S), torch.uint8),
            ("mu", (B,), torch.float64), ("sigma", (B, B), torch.float64),
            ("inv", (B, B), torch.float64), ("chol", (B, B), torch.float64),
            ("ridge", (1,), torch.float64), ("status", (1,), torch.int32),
            ("flags", (1,), torch.int32), ("thr", (1,), torch.float32),
            ("key", (1,), torch.int32))}
        ds = plan.ds
        with torch.cuda.stream(copy):
            copy.wait_event(comp_done[i])
            for name, t in (("scores", plan.scores[j]), ("mask", plan.mask[j]),
                            ("mu", ds.mu[j]), ("sigma", ds.sigma[j]), ("inv", ds.sigma_inv[j]),
                            ("chol", ds.chol[j]), ("ridge", ds.ridge[j:j + 1]),
                            ("status", ds.status[j:j + 1]), ("flags", ds.flags[j:j + 1]),
                            ("thr", plan.thr[j:j + 1]),
                            ("key", plan.max_key[j:j + 1].view(torch.int32))):
                o[name].copy_(t, non_blocking=True)
            d2h.append(ev())
            d2h[i].record(copy)
        outs.append(o)
    copy.synchronize()
    comp.synchronize()
    dets = []
    for i, o in enumerate(outs):
        st, fl = int(o["status"][0]), int(o["flags"][0])
        if st == _lib.ERR_RANGE or fl & 48:
            dets.append(detect(raws[i], tabs[i], k=k, device=False))  # general path
            continue
        if st == _lib.ERR_INSUFFICIENT:
            raise ValueError(f"insufficient samples: {n} pixels for {B} bands")
        if st != _lib.OK:
            raise ValueError(_STATUS_MSG.get(st, f"stats failed with status {st}"))
        stats = CubeStats(mu=o["mu"].numpy(), sigma=o["sigma"].numpy(),
                          sigma_inv=o["inv"].numpy(), ridge_used=float(o["ridge"][0]),
                          chol_lower=o["chol"].numpy())
        key = torch.tensor([int(o["key"][0]) & 0xFFFFFFFF])
        dets.append(Detection(stats, o["scores"].numpy(), o["mask"].numpy().view(bool),
                              float(o["thr"][0]), key_to_float(key)))
    return dets
