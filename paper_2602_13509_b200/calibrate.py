"""Radiometric calibration on the B200 — drop-in for skyrx.calibrate.

Same names, arguments, return types and error messages as the reference
(calibrate.py:32-176); the arithmetic runs in the K1 CUDA kernels
(csrc/calibrate.cu) and is bit-identical to the reference:

    radiance[l, s, b] = max(0, raw[l, s, b] - dark[s, b]) * coeff[s, b] / gain[l]

Host (numpy) cubes are copied to the device and results copied back; CUDA
tensors stay on the device.  `.hsk` table file I/O (calibrate.py:56-80) is
disk plumbing and out of scope.
"""

from __future__ import annotations

import sys
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev, _lib
from .cube import RadianceCube, band_nearest

BAND_KEEP_MIN_NM = 400.0
BAND_KEEP_MAX_NM = 1000.0
RGB_TARGETS_NM = (640.0, 550.0, 460.0)


@dataclass(frozen=True)
class CalibrationTables:
    """calibrate.py:32-53: per-(sample, band) dark offsets and coefficients (f32)."""

    dark: np.ndarray
    coeff: np.ndarray
    _cache: dict = field(default_factory=dict, compare=False, repr=False)
    _lock: object = field(default_factory=threading.Lock, compare=False, repr=False)

    def __post_init__(self):
        object.__setattr__(self, "dark", np.ascontiguousarray(self.dark, dtype=np.float32))
        object.__setattr__(self, "coeff", np.ascontiguousarray(self.coeff, dtype=np.float32))
        if self.dark.shape != self.coeff.shape or self.dark.ndim != 2:
            raise ValueError("dark and coeff must be equal-shaped 2-D grids")
        if not (self.coeff > 0).all():
            raise ValueError("coeff must be positive everywhere")

    @property
    def samples(self) -> int:
        return self.dark.shape[0]

    @property
    def bands(self) -> int:
        return self.dark.shape[1]

    def device(self):
        """(dark, coeff) as device tensors, uploaded once per device."""
        dev = _dev.require_cuda()
        with self._lock:
            hit = self._cache.get(dev.index)
            if hit is None:
                hit = (_dev.to_device(self.dark), _dev.to_device(self.coeff))
                self._cache[dev.index] = hit
        return hit


def tables_of(tables):
    """Accept our CalibrationTables or the reference's (duck-typed)."""
    if isinstance(tables, CalibrationTables):
        return tables
    return CalibrationTables(tables.dark, tables.coeff)


def _out_cls(obj, name, default):
    mod = sys.modules.get(type(obj).__module__, None)
    if mod is not None and mod.__name__.startswith("skyrx") and not _dev.is_device(obj.values):
        return getattr(mod, name, default)
    return default


def line_gains(cube):
    """calibrate.py:83-87: per-line gains as f32; all must be > 0."""
    g = getattr(cube, "gains", None)
    if g is None:
        g = np.array([m.gain for m in cube.line_meta], dtype=np.float32)
    if isinstance(g, torch.Tensor):
        g = g.to(torch.float32)
        if g.numel() and not bool((g > 0).all()):
            raise ValueError("every line gain must be positive")
        return g
    g = np.asarray(g, dtype=np.float32)
    if not (g > 0).all():
        raise ValueError("every line gain must be positive")
    return g


def _check_tables(raw, tables):
    if (tables.samples, tables.bands) != (raw.samples, raw.bands):
        raise ValueError(
            f"invalid tables: shape ({tables.samples}, {tables.bands}) does not "
            f"match cube ({raw.samples}, {raw.bands})"
        )


def _raw_device(raw):
    v = raw.values
    if isinstance(v, torch.Tensor):
        if v.dtype not in (torch.uint16, torch.int16):
            v = v.to(torch.int32).to(torch.uint16)
        return _dev.to_device(v.view(torch.uint16) if v.dtype == torch.int16 else v)
    return _dev.to_device(np.asarray(v), torch.uint16)


def apply_calibration(raw, tables) -> RadianceCube:
    """Convert raw digital numbers to gain-independent radiance (calibrate.py:90-102)."""
    tables = tables_of(tables)
    _check_tables(raw, tables)
    gains = line_gains(raw)
    if len(gains) != raw.lines:
        raise ValueError(f"line_meta: {len(gains)} gains for {raw.lines} lines")
    dark, coeff = tables.device()
    rv = _raw_device(raw)
    gd = _dev.to_device(gains, torch.float32)
    out = _dev.empty((raw.lines, raw.samples, raw.bands), torch.float32)
    _lib.call("skyrx_calibrate", rv.data_ptr(), raw.lines, raw.samples, raw.bands,
              dark.data_ptr(), coeff.data_ptr(), gd.data_ptr(), None, 0, 1, out.data_ptr(),
              None, None, _dev.stream_ptr())
    cls = _out_cls(raw, "RadianceCube", RadianceCube)
    return cls(_dev.like_input(raw.values, out), raw.wavelengths_nm, raw.line_meta)


def _keep_index(wavelengths) -> np.ndarray:
    w = np.asarray(wavelengths, dtype=np.float64)
    return np.nonzero((w >= BAND_KEEP_MIN_NM) & (w <= BAND_KEEP_MAX_NM))[0].astype(np.int32)


def _rebin(cube, keep, factor, rgb_idx=None):
    values = _dev.to_device(cube.values, torch.float32)
    L, S, B = cube.lines, cube.samples, cube.bands
    nout = len(keep) // factor
    out = _dev.empty((L, S, nout), torch.float32)
    rgb = _dev.empty((L, S, 3), torch.float32) if rgb_idx is not None else None
    kd = _dev.to_device(keep, torch.int32) if len(keep) else None
    ridx = (np.asarray(rgb_idx, np.int32).ctypes.data_as(_lib.C.POINTER(_lib.C.c_int32))
            if rgb_idx is not None else None)
    if L * S and nout:
        _lib.call("skyrx_bin_radiance", values.data_ptr(), L, S, B, _dev.ptr(kd), len(keep),
                  factor, out.data_ptr(), ridx, _dev.ptr(rgb), _dev.stream_ptr())
    return out, rgb


def discard_oob_bands(cube) -> RadianceCube:
    """calibrate.py:105-114: drop band centres outside [400, 1000] nm."""
    keep = _keep_index(cube.wavelengths_nm)
    out, _ = _rebin(cube, keep, 1)
    cls = _out_cls(cube, "RadianceCube", RadianceCube)
    return cls(_dev.like_input(cube.values, out), cube.wavelengths_nm[keep], cube.line_meta)


def bin_bands(cube, factor: int = 4) -> RadianceCube:
    """calibrate.py:117-126: sum each run of ``factor`` bands (f32, left to right)."""
    if factor < 1 or cube.bands % factor != 0:
        raise ValueError(f"band count {cube.bands} not divisible by factor {factor}")
    out_bands = cube.bands // factor
    out, _ = _rebin(cube, np.arange(cube.bands, dtype=np.int32), factor)
    centers = np.asarray(cube.wavelengths_nm).reshape(out_bands, factor).mean(axis=1)
    cls = _out_cls(cube, "RadianceCube", RadianceCube)
    return cls(_dev.like_input(cube.values, out), centers, cube.line_meta)


def extract_rgb(cube):
    """calibrate.py:129-132: (lines, samples, 3) planes nearest 640/550/460 nm."""
    idx = np.array([band_nearest(cube.wavelengths_nm, t) for t in RGB_TARGETS_NM], np.int32)
    out, _ = _rebin(cube, idx, 1)
    return _dev.like_input(cube.values, out)


def calibrate_bin_rgb(raw, tables, factor: int = 4, chunk_lines: int = 64):
    """calibrate.py:135-176: fused calibrate -> discard -> bin -> RGB in one kernel.

    ``chunk_lines`` is accepted for signature compatibility; the device kernel
    streams the whole cube and never materialises the full-band radiance.
    """
    tables = tables_of(tables)
    _check_tables(raw, tables)
    gains = line_gains(raw)
    keep = _keep_index(raw.wavelengths_nm)
    kept = len(keep)
    if factor < 1 or kept % factor != 0:
        raise ValueError(f"band count {kept} not divisible by factor {factor}")
    out_bands = kept // factor
    centers = np.asarray(raw.wavelengths_nm)[keep].reshape(out_bands, factor).mean(axis=1)
    rgb_idx = np.array([band_nearest(centers, t) for t in RGB_TARGETS_NM], np.int32)
    dark, coeff = tables.device()
    rv = _raw_device(raw)
    gd = _dev.to_device(gains, torch.float32)
    L, S = raw.lines, raw.samples
    out = _dev.empty((L, S, out_bands), torch.float32)
    rgb = _dev.empty((L, S, 3), torch.float32)
    if L * S and out_bands:
        kd = _dev.to_device(keep, torch.int32)
        _lib.call("skyrx_calibrate", rv.data_ptr(), L, S, raw.bands, dark.data_ptr(),
                  coeff.data_ptr(), gd.data_ptr(), kd.data_ptr(), kept, factor, out.data_ptr(),
                  rgb_idx.ctypes.data_as(_lib.C.POINTER(_lib.C.c_int32)), rgb.data_ptr(),
                  _dev.stream_ptr())
    cls = _out_cls(raw, "RadianceCube", RadianceCube)
    binned = cls(_dev.like_input(raw.values, out), centers, raw.line_meta)
    return binned, _dev.like_input(raw.values, rgb)
