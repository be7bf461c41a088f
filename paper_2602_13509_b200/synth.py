"""Device-side seeded synthetic raw cubes (bench and large-shape test inputs).

Wraps ``skyrx_synth_raw`` (csrc/synth.cu).  The scene/sensor parameter
tables are small and built on the host by the frozen recipe in
``SceneSpec.tables`` (identical numbers to oracle/synth.py make_tables, which
the tests check); the per-element hashing and f32 arithmetic run on the GPU
and are bit-identical to oracle/synth.py generate_lines.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _lib

R_LATENT = 6
N_ANOMALY_SPECTRA = 32
M32 = 0xFFFFFFFF


def _fmix32(h: int) -> int:
    h &= M32
    h ^= h >> 16
    h = (h * 0x85EBCA6B) & M32
    h ^= h >> 13
    h = (h * 0xC2B2AE35) & M32
    h ^= h >> 16
    return h


def seed_keys(seed: int) -> tuple[int, int]:
    sk = _fmix32((seed * 0x9E3779B9 + 0x632BE5AB) & M32)
    return sk, _fmix32(sk ^ 0xA511E9B3)


def _smooth(rng, bands, terms, amp):
    b = np.arange(bands, dtype=np.float64) / max(bands - 1, 1)
    out = np.zeros(bands)
    for j in range(1, terms + 1):
        out += rng.uniform(-amp, amp) / j * np.cos(np.pi * j * b + rng.uniform(0, 2 * np.pi))
    return out


class Scene:
    """Seeded scene + sensor for (seed, samples, bands, components)."""

    def __init__(self, seed: int, samples: int, bands: int, components: int = 5):
        self.seed, self.samples, self.bands, self.components = seed, samples, bands, components
        rng = np.random.default_rng([seed, samples, bands, components])
        k = components
        w = rng.dirichlet(np.full(k, 2.0))
        self.cw24 = np.floor(np.cumsum(w)[:-1] * (1 << 24)).astype(np.uint32)
        levels = rng.uniform(900.0, 2200.0, k)
        mean = np.stack([levels[i] * (1.0 + _smooth(rng, bands, 4, 0.25)) for i in range(k)])
        factor = np.zeros((k, bands, R_LATENT))
        for i in range(k):
            for j in range(R_LATENT):
                factor[i, :, j] = levels[i] * 0.03 / np.sqrt(R_LATENT) * (
                    rng.uniform(0.5, 1.5) + _smooth(rng, bands, 3, 1.0))
        sd = levels[:, None] * rng.uniform(0.003, 0.01, (k, bands))
        alev = rng.uniform(900.0, 2600.0, N_ANOMALY_SPECTRA)
        aspec = np.stack([alev[i] * (1.0 + _smooth(rng, bands, 6, 0.5))
                          for i in range(N_ANOMALY_SPECTRA)])
        aspec = np.clip(aspec, 50.0, None)
        asd = np.full(bands, 0.005 * levels.mean())
        xbar = mean.mean(axis=0)
        dark = rng.normal(100.0, 3.0, (samples, bands)).astype(np.float32)
        white = 3500.0 * (1.0 + rng.uniform(-0.1, 0.1, (samples, bands)))
        coeff = (np.float32(3400.0) / (white.astype(np.float32) - dark)).astype(np.float32)
        f = lambda a: np.ascontiguousarray(a, dtype=np.float32)  # noqa: E731
        self.mean, self.factor, self.sd = f(mean), f(factor), f(sd)
        self.aspec, self.asd, self.xbar = f(aspec), f(asd), f(xbar)
        self.dark, self.coeff = dark, coeff
        self.seedkey, self.cellkey = seed_keys(seed)
        self._dev = None

    def _device_tables(self):
        if self._dev is None:
            self._dev = {name: _dev.to_device(getattr(self, name)) for name in
                         ("cw24", "mean", "factor", "sd", "aspec", "asd", "xbar", "dark",
                          "coeff")}
        return self._dev

    def generate(self, line0: int, nlines: int, out: torch.Tensor | None = None) -> torch.Tensor:
        """Raw uint16 (nlines, samples, bands) on the current CUDA device."""
        t = self._device_tables()
        if out is None:
            out = _dev.empty((nlines, self.samples, self.bands), torch.uint16)
        if self.components > 1:
            cw = t["cw24"].data_ptr()
        else:
            cw = _dev.zeros((1,), torch.uint32).data_ptr()
        _lib.call("skyrx_synth_raw", self.seedkey, self.cellkey, self.samples, self.bands,
                  self.components, cw, t["mean"].data_ptr(), t["factor"].data_ptr(),
                  t["sd"].data_ptr(), t["aspec"].data_ptr(), t["asd"].data_ptr(),
                  t["xbar"].data_ptr(), t["dark"].data_ptr(), t["coeff"].data_ptr(), line0,
                  nlines, out.data_ptr(), _dev.stream_ptr())
        return out
