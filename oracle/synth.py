"""Seeded synthetic push-broom raw cubes — CPU twin of the device generator.

TEST INFRASTRUCTURE (oracle/): only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs import this module.  The
product path never does.

Why this exists
---------------
BASELINE.json's configs describe seeded synthetic cubes (K-component Gaussian
mixture background, smooth random spectra, 2% Poisson-like noise, 0.1% of
pixels planted as 3x3..8x8 anomaly blobs, dark ~ N(100, 3), white = 3500 with
+/-10% response).  The paper's Memphis flights are not available, so these
stand in for them.  The reference's own generator
(`skyrx/scene.py:254-361`, raw digitisation `scene.py:348-357`) draws with
numpy's sequential RNG, which cannot be regenerated block-by-block on a GPU.
This generator is counter-based instead: every raw count is a pure function of
(seed, line, sample, band) built from 32-bit integer hashing and individually
rounded IEEE float32 operations (+, *, /, sqrt, rint - all correctly rounded
in numpy and in CUDA without fast-math).  The CUDA kernel
`skyrx_synth_raw` (csrc/synth.cu) performs the same operations in the same
order, so any line block of any config is bit-identical on CPU and GPU, which
lets parity tests run on cubes far larger than the oracle could generate
in one go.

Frozen definition (changing anything here changes every golden number):
    pixel key   pk = fmix32(g_lo ^ fmix32(g_hi ^ seedkey)),  g = line*S + sample
    stream hash Hs(pk, j)    = fmix32(pk + j * 0x9E3779B9)
    band hash   Hb(pk, b, j) = fmix32(pk ^ (b * 0x85EBCA77 + j * 0xC2B2AE3D))
    IH4(h)      = (sum of the 4 bytes of h - 510) * f32(1/sqrt(21845))  (approx N(0,1))
    component   k = #{cw[i] <= Hs(pk,0) >> 8}
    latent      g_j = IH4(Hs(pk, 1+j)), j < R
    band noise  n1 = IH4(Hb(pk,b,1)), n2 = IH4(Hb(pk,b,2))
    background  t = M[k,b]; t += A[k,b,j]*g_j (j ascending); t += SD[k,b]*n1
    anomaly     t = AS[a,b] + ASD[b]*n1   (pixel inside a planted blob)
    both        t = max(t,0); q = sqrt(t*XBAR[b]) * 0.02; t += q*n2
    raw         clip(rint(t / COEFF[s,b] + DARK[s,b]), 0, 4095) -> uint16
Anomaly blobs live on a 16x16-pixel cell grid: a cell holds one square blob
(side U{3..8}, random offset inside the cell, spectrum a = one of NA) with
probability p chosen so that the expected anomalous fraction is 0.1%.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

R_LATENT = 6          # rank of the smooth per-component covariance factor
N_ANOMALY_SPECTRA = 32
CELL = 16             # anomaly cell edge (pixels)
ANOMALY_FRACTION = 0.001
_E_SIDE2 = sum(s * s for s in range(3, 9)) / 6.0
P_CELL24 = int(round(ANOMALY_FRACTION * CELL * CELL / _E_SIDE2 * (1 << 24)))
INV_IH4 = np.float32(1.0 / np.sqrt(4.0 * (256.0 * 256.0 - 1.0) / 12.0))
NOISE_FRAC = np.float32(0.02)
RAW_MAX = 4095.0

M32 = 0xFFFFFFFF


def _fmix32_int(h: int) -> int:
    h &= M32
    h ^= h >> 16
    h = (h * 0x85EBCA6B) & M32
    h ^= h >> 13
    h = (h * 0xC2B2AE35) & M32
    h ^= h >> 16
    return h


def fmix32(h: np.ndarray) -> np.ndarray:
    """murmur3 finaliser on uint32 arrays (wrapping arithmetic)."""
    h = np.asarray(h, dtype=np.uint32)
    h = h ^ (h >> np.uint32(16))
    h = h * np.uint32(0x85EBCA6B)
    h = h ^ (h >> np.uint32(13))
    h = h * np.uint32(0xC2B2AE35)
    h = h ^ (h >> np.uint32(16))
    return h


def seed_key(seed: int) -> int:
    return _fmix32_int((seed * 0x9E3779B9 + 0x632BE5AB) & M32)


def cell_seed_key(seed: int) -> int:
    return _fmix32_int(seed_key(seed) ^ 0xA511E9B3)


def ih4(h: np.ndarray) -> np.ndarray:
    h = h.astype(np.uint32)
    s = (
        (h & np.uint32(255)).astype(np.int32)
        + ((h >> np.uint32(8)) & np.uint32(255)).astype(np.int32)
        + ((h >> np.uint32(16)) & np.uint32(255)).astype(np.int32)
        + (h >> np.uint32(24)).astype(np.int32)
        - 510
    )
    return s.astype(np.float32) * INV_IH4


@dataclass(frozen=True)
class SceneTables:
    """Host-side parameters of one seeded scene + sensor (all float32)."""

    seed: int
    samples: int
    bands: int
    components: int
    cw24: np.ndarray     # (K-1,) uint32 cumulative component thresholds in [0, 2^24]
    mean: np.ndarray     # (K, B)
    factor: np.ndarray   # (K, B, R)
    sd: np.ndarray       # (K, B)
    aspec: np.ndarray    # (NA, B)
    asd: np.ndarray      # (B,)
    xbar: np.ndarray     # (B,)
    dark: np.ndarray     # (S, B)
    coeff: np.ndarray    # (S, B)

    @property
    def seedkey(self) -> int:
        return seed_key(self.seed)

    @property
    def cellkey(self) -> int:
        return cell_seed_key(self.seed)


def _smooth(rng, bands, terms, amp):
    b = np.arange(bands, dtype=np.float64) / max(bands - 1, 1)
    out = np.zeros(bands)
    for j in range(1, terms + 1):
        out += rng.uniform(-amp, amp) / j * np.cos(np.pi * j * b + rng.uniform(0, 2 * np.pi))
    return out


def make_tables(seed: int, samples: int, bands: int, components: int = 5) -> SceneTables:
    """Deterministic scene/sensor parameters for (seed, samples, bands, K)."""
    rng = np.random.default_rng([seed, samples, bands, components])
    k = components
    w = rng.dirichlet(np.full(k, 2.0))
    cw = np.floor(np.cumsum(w)[:-1] * (1 << 24)).astype(np.uint32)
    levels = rng.uniform(900.0, 2200.0, k)
    mean = np.stack([levels[i] * (1.0 + _smooth(rng, bands, 4, 0.25)) for i in range(k)])
    factor = np.zeros((k, bands, R_LATENT))
    for i in range(k):
        for j in range(R_LATENT):
            factor[i, :, j] = levels[i] * 0.03 / np.sqrt(R_LATENT) * (
                rng.uniform(0.5, 1.5) + _smooth(rng, bands, 3, 1.0)
            )
    sd = levels[:, None] * rng.uniform(0.003, 0.01, (k, bands))
    alevels = rng.uniform(900.0, 2600.0, N_ANOMALY_SPECTRA)
    aspec = np.stack(
        [alevels[i] * (1.0 + _smooth(rng, bands, 6, 0.5)) for i in range(N_ANOMALY_SPECTRA)]
    )
    aspec = np.clip(aspec, 50.0, None)
    asd = np.full(bands, 0.005 * levels.mean())
    xbar = mean.mean(axis=0)
    dark = rng.normal(100.0, 3.0, (samples, bands))
    white = 3500.0 * (1.0 + rng.uniform(-0.1, 0.1, (samples, bands)))
    dark32 = dark.astype(np.float32)
    coeff = (np.float32(3400.0) / (white.astype(np.float32) - dark32)).astype(np.float32)
    f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)  # noqa: E731
    return SceneTables(
        seed=seed, samples=samples, bands=bands, components=k, cw24=cw,
        mean=f32(mean), factor=f32(factor), sd=f32(sd), aspec=f32(aspec),
        asd=f32(asd), xbar=f32(xbar), dark=dark32, coeff=f32(coeff),
    )


def _pixel_keys(seedkey: int, g: np.ndarray) -> np.ndarray:
    g = g.astype(np.uint64)
    lo = (g & np.uint64(M32)).astype(np.uint32)
    hi = (g >> np.uint64(32)).astype(np.uint32)
    return fmix32(lo ^ fmix32(hi ^ np.uint32(seedkey)))


def anomaly_index(tables: SceneTables, lines: np.ndarray, samples: np.ndarray) -> np.ndarray:
    """Anomaly spectrum index per pixel, -1 where the pixel is background."""
    l = lines.astype(np.int64)
    s = samples.astype(np.int64)
    ncs = (tables.samples + CELL - 1) // CELL
    cell = ((l // CELL) * ncs + (s // CELL)).astype(np.uint64)
    ck = fmix32((cell & np.uint64(M32)).astype(np.uint32) ^ np.uint32(tables.cellkey))
    present = (ck >> np.uint32(8)) < np.uint32(P_CELL24)
    h2 = fmix32(ck + np.uint32(0x68E31DA4))
    side = (h2 % np.uint32(6)).astype(np.int64) + 3
    span = 17 - side
    ol = ((h2 >> np.uint32(8)).astype(np.int64)) % span
    os_ = ((h2 >> np.uint32(16)).astype(np.int64)) % span
    a = ((h2 >> np.uint32(24)).astype(np.int64)) % N_ANOMALY_SPECTRA
    dl = (l % CELL) - ol
    ds = (s % CELL) - os_
    inside = present & (dl >= 0) & (dl < side) & (ds >= 0) & (ds < side)
    return np.where(inside, a, -1)


def generate_lines(tables: SceneTables, line0: int, nlines: int) -> np.ndarray:
    """Raw uint16 counts for lines [line0, line0+nlines), shape (nlines, S, B)."""
    S, B = tables.samples, tables.bands
    out = np.empty((nlines, S, B), dtype=np.uint16)
    step = max(1, (1 << 22) // max(S * B, 1))
    b = np.arange(B, dtype=np.uint32)
    for c0 in range(0, nlines, step):
        c1 = min(nlines, c0 + step)
        ll = np.arange(line0 + c0, line0 + c1, dtype=np.int64)
        lg, sg = np.meshgrid(ll, np.arange(S, dtype=np.int64), indexing="ij")
        lg, sg = lg.ravel(), sg.ravel()
        g = lg * S + sg
        pk = _pixel_keys(tables.seedkey, g)
        hs0 = fmix32(pk)  # Hs(pk, 0)
        comp = np.searchsorted(tables.cw24, hs0 >> np.uint32(8), side="right")
        t = tables.mean[comp]                                        # (P, B)
        for j in range(R_LATENT):
            gj = ih4(fmix32(pk + np.uint32((1 + j) * 0x9E3779B9 & M32)))
            t = t + tables.factor[comp, :, j] * gj[:, None]
        hb1 = fmix32(pk[:, None] ^ (b[None, :] * np.uint32(0x85EBCA77) + np.uint32(0xC2B2AE3D)))
        n1 = ih4(hb1)
        t = t + tables.sd[comp] * n1
        aidx = anomaly_index(tables, lg, sg)
        hit = aidx >= 0
        if hit.any():
            ta = tables.aspec[aidx[hit]] + tables.asd[None, :] * n1[hit]
            t[hit] = ta
        t = np.maximum(t, np.float32(0.0))
        hb2 = fmix32(pk[:, None] ^ (b[None, :] * np.uint32(0x85EBCA77) + np.uint32(2 * 0xC2B2AE3D & M32)))
        n2 = ih4(hb2)
        q = t * tables.xbar[None, :]
        q = np.sqrt(q)
        q = q * NOISE_FRAC
        t = t + q * n2
        dn = t / tables.coeff[sg] + tables.dark[sg]
        dn = np.rint(dn)
        dn = np.clip(dn, np.float32(0.0), np.float32(RAW_MAX))
        out[c0:c1] = dn.astype(np.uint16).reshape(c1 - c0, S, B)
    return out


def anomaly_mask(tables: SceneTables, line0: int, nlines: int) -> np.ndarray:
    ll = np.arange(line0, line0 + nlines, dtype=np.int64)
    lg, sg = np.meshgrid(ll, np.arange(tables.samples, dtype=np.int64), indexing="ij")
    return anomaly_index(tables, lg, sg) >= 0


# BASELINE.json configs; lines, samples, bands, components, seed
CONFIGS = {
    "c1": dict(lines=2048, samples=900, bands=70, components=5, seed=1),
    "c2": dict(lines=60 * 249, samples=900, bands=70, components=5, seed=2, chunk_lines=249,
               forget=0.99),
    "c3": dict(lines=8192, samples=1024, bands=270, components=8, seed=3),
    "c4": dict(lines=16384, samples=900, bands=70, components=5, seed=4000, strips=64),
    "c5": dict(lines=131072, samples=2048, bands=128, components=5, seed=5),
}
