"""The reference's kernel slot, served by the B200 library.

skyrx._accel (_accel.py:19-131) picks numba or numpy at import time and
exposes ``mahalanobis_sq(pixels, mu, chol_lower) -> (N,) float64``; rx_scores
looks it up at call time (rx.py:20, 96).  This module exposes the same name
backed by ``skyrx_mahalanobis_sq`` (FP64 whitening product on the GPU), so
``install()`` can drop it into the reference unchanged.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev
from .rx import mahalanobis_sq_device

HAS_NUMBA = False   # attribute kept for drop-in compatibility (_accel.py:24-30)
HAS_CUDA = True


def mahalanobis_sq(pixels, mu, chol_lower):
    """Squared Mahalanobis distance per row of ``pixels`` (N, B), float64."""
    if _dev.is_device(pixels):
        return mahalanobis_sq_device(pixels, mu, chol_lower)
    px = np.ascontiguousarray(pixels)
    if px.dtype not in (np.float32, np.float64):
        px = px.astype(np.float64)
    d = mahalanobis_sq_device(_dev.to_device(px), np.asarray(mu, np.float64),
                              np.asarray(chol_lower, np.float64))
    return _dev.to_host(d)


def mahalanobis_sq_numpy(pixels, mu, chol_lower, chunk: int = 65536):
    """Name kept for drop-in compatibility; runs the same device kernel."""
    return mahalanobis_sq(pixels, mu, chol_lower)


__all__ = ["HAS_NUMBA", "HAS_CUDA", "mahalanobis_sq", "mahalanobis_sq_numpy", "torch"]
