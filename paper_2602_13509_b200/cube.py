"""Boundary data model, mirroring skyrx.cube (cube.py:28-258).

Same names, fields and invariants as the reference so the parity tests read
like the reference's own.  Differences, all additive:
  * ``values`` may be a CUDA ``torch.Tensor`` (device-resident fast path,
    no host copies) as well as a numpy array;
  * ``RawCube`` accepts an optional ``gains`` array so very long strips do not
    need one ``LineMeta`` object per line (the reference derives gains from
    ``line_meta``, calibrate.py:83-87; both routes give identical f32 gains).
Every API function also accepts the reference's own ``skyrx.cube`` objects
(duck-typed on ``values`` / ``wavelengths_nm`` / ``line_meta``).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence, Union

import numpy as np

try:  # torch is the device allocator; the data model itself does not need it
    import torch
except ImportError:  # pragma: no cover
    torch = None


def _is_tensor(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor)


def _as_values(v, dtype=None):
    if _is_tensor(v):
        return v
    return np.asarray(v) if dtype is None else np.asarray(v, dtype=dtype)


@dataclass(frozen=True)
class InsSample:
    """cube.py:28-41."""

    timestamp_us: int
    lat_deg: float
    lon_deg: float
    alt_m: float
    roll_deg: float
    pitch_deg: float
    yaw_deg: float


@dataclass(frozen=True)
class LineMeta:
    """cube.py:44-51: per-line exposure start, gain and bracketing INS."""

    exposure_start_us: int
    gain: float
    ins_before: InsSample
    ins_after: InsSample


@dataclass(frozen=True, eq=False)
class RawCube:
    """cube.py:80-105: uint16 (lines, samples, bands), bands innermost."""

    values: object
    wavelengths_nm: np.ndarray
    line_meta: tuple = ()
    gains: object = field(default=None)

    def __post_init__(self):
        object.__setattr__(self, "values", _as_values(self.values))
        object.__setattr__(self, "wavelengths_nm",
                           np.asarray(self.wavelengths_nm, dtype=np.float64))
        object.__setattr__(self, "line_meta", tuple(self.line_meta))

    @property
    def lines(self) -> int:
        return int(self.values.shape[0])

    @property
    def samples(self) -> int:
        return int(self.values.shape[1])

    @property
    def bands(self) -> int:
        return int(self.values.shape[2])


@dataclass(frozen=True, eq=False)
class RadianceCube:
    """cube.py:108-137: float32 calibrated cube."""

    values: object
    wavelengths_nm: np.ndarray
    line_meta: tuple = ()

    def __post_init__(self):
        object.__setattr__(self, "values", _as_values(self.values, np.float32)
                           if not _is_tensor(self.values) else self.values)
        object.__setattr__(self, "wavelengths_nm",
                           np.asarray(self.wavelengths_nm, dtype=np.float64))
        object.__setattr__(self, "line_meta", tuple(self.line_meta))

    @property
    def lines(self) -> int:
        return int(self.values.shape[0])

    @property
    def samples(self) -> int:
        return int(self.values.shape[1])

    @property
    def bands(self) -> int:
        return int(self.values.shape[2])


Cube = Union[RawCube, RadianceCube]


@dataclass(frozen=True, eq=False)
class GroundTruthMask:
    """cube.py:140-158."""

    values: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "values", np.asarray(self.values, dtype=bool))


@dataclass(frozen=True, eq=False)
class ScoreMap:
    """cube.py:161-184: per-pixel scores; ``max_score`` is the grid maximum."""

    values: object

    def __post_init__(self):
        if not _is_tensor(self.values):
            object.__setattr__(self, "values", np.asarray(self.values, dtype=np.float32))

    @property
    def max_score(self) -> float:
        v = self.values
        if _is_tensor(v):
            return float(v.max().item()) if v.numel() else 0.0
        return float(v.max()) if v.size else 0.0

    @property
    def lines(self) -> int:
        return int(self.values.shape[0])

    @property
    def samples(self) -> int:
        return int(self.values.shape[1])


def band_nearest(wavelengths_nm: Sequence[float], target_nm: float) -> int:
    """cube.py:187-195: nearest band centre, ties to the lower index."""
    ws = np.asarray(wavelengths_nm, dtype=np.float64)
    if ws.size == 0:
        raise ValueError("wavelength list is empty")
    return int(np.argmin(np.abs(ws - target_nm)))


def line_meta_for(gains) -> tuple:
    """Convenience: LineMeta records for a gain vector (synthetic cubes)."""
    out = []
    t0 = 1_600_000_000_000_000
    for i, g in enumerate(np.asarray(gains, dtype=np.float64).tolist()):
        t = t0 + i * 4016
        ins = InsSample(t - 1000, 0.0, 0.0, 40.0, 0.0, 0.0, 0.0)
        ins2 = InsSample(t + 4000, 0.0, 0.0, 40.0, 0.0, 0.0, 0.0)
        out.append(LineMeta(t, g, ins, ins2))
    return tuple(out)
