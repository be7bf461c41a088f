"""CPU restatement of the reference's calibrate + RX hot path (numpy / LAPACK).

TEST INFRASTRUCTURE (oracle/): this module is the *checker*.  Only tests/,
``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` / ``--impl
reference`` legs may import it.  The product (paper_2602_13509_b200) never
routes through it; its ops fail loudly when the CUDA library is missing.

Each function restates one reference function over plain arrays and cites the
reference line it follows (paths relative to /root/reference/pkg/src/skyrx).
Pinned against the reference itself: tests/golden/*.npz were produced by
importing the real `skyrx` package (tests/golden/make_golden.py) and
tests/test_oracle.py checks this module against every fixture.

Three rows of SURVEY.md §8(a) have no reference implementation; their frozen
definitions live here (R-TOPK ``topk_threshold``/``topk_mask``, R-STREAM
``StreamingStats``, R-GLOBAL ``moments``/``combine_moments``/``finalize_moments``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.linalg import cho_solve, solve_triangular

# rx.py:23 — diagonal-loading ladder tried after the unridged attempt
RIDGE_EPSILONS = (1e-10, 1e-9, 1e-8, 1e-7, 1e-6)
BAND_KEEP_MIN_NM = 400.0   # calibrate.py:23
BAND_KEEP_MAX_NM = 1000.0  # calibrate.py:24
RGB_TARGETS_NM = (640.0, 550.0, 460.0)  # calibrate.py:25


# --------------------------------------------------------------------------- calibration
def line_gains(gains) -> np.ndarray:
    """calibrate.py:83-87 — per-line gains as float32, all strictly positive."""
    g = np.asarray(gains, dtype=np.float32)
    if not (g > 0).all():
        raise ValueError("every line gain must be positive")
    return g


def _check_tables(shape, dark, coeff):
    # calibrate.py:92-96 / 150-154
    if tuple(dark.shape) != (shape[1], shape[2]):
        raise ValueError(
            f"invalid tables: shape ({dark.shape[0]}, {dark.shape[1]}) does not "
            f"match cube ({shape[1]}, {shape[2]})"
        )


def apply_calibration(raw, dark, coeff, gains) -> np.ndarray:
    """calibrate.py:90-102: max(0, f32(raw) - dark) * coeff / gain[l], each op f32 RN."""
    raw = np.asarray(raw)
    dark = np.asarray(dark, np.float32)
    coeff = np.asarray(coeff, np.float32)
    _check_tables(raw.shape, dark, coeff)
    g = line_gains(gains)
    x = raw.astype(np.float32) - dark[None]
    np.maximum(x, np.float32(0.0), out=x)
    x *= coeff[None]
    x /= g[:, None, None]
    return x


def keep_bands(wavelengths) -> np.ndarray:
    """calibrate.py:105-114 — boolean keep mask for centres in [400, 1000] nm."""
    w = np.asarray(wavelengths, dtype=np.float64)
    return (w >= BAND_KEEP_MIN_NM) & (w <= BAND_KEEP_MAX_NM)


def band_nearest(wavelengths, target) -> int:
    """cube.py:187-195 — argmin |w - target|, ties to the lower index."""
    w = np.asarray(wavelengths, dtype=np.float64)
    if w.size == 0:
        raise ValueError("wavelength list is empty")
    return int(np.argmin(np.abs(w - target)))


def sequential_sum_f32(x: np.ndarray) -> np.ndarray:
    """Last-axis f32 sum, strictly left to right: ((a0+a1)+a2)+...

    This is the order the reference actually gets at calibrate.py:173 (and
    bin_bands, calibrate.py:122-124): ``block[:, :, keep]`` is a boolean index
    on the last axis, which numpy materialises band-major (strides
    (S*4, 4, L*S*4)), so the reduction over each group of ``factor`` bands
    accumulates one band at a time for every factor.  Verified bit-exact
    against the reference for factor 4 and 8 (tests/test_oracle.py)."""
    x = np.asarray(x, np.float32)
    acc = x[..., 0].copy()
    for j in range(1, x.shape[-1]):
        acc += x[..., j]
    return acc


def binned_centers(wavelengths, factor):
    keep = keep_bands(wavelengths)
    kept = int(keep.sum())
    if factor < 1 or kept % factor != 0:
        raise ValueError(f"band count {kept} not divisible by factor {factor}")
    return np.asarray(wavelengths, np.float64)[keep].reshape(kept // factor, factor).mean(axis=1)


def calibrate_bin_rgb(raw, wavelengths, dark, coeff, gains, factor=4, chunk_lines=64):
    """calibrate.py:135-176 — calibrate, drop out-of-range bands, sum ``factor``
    consecutive bands left to right in f32, then pick RGB planes."""
    raw = np.asarray(raw)
    dark = np.asarray(dark, np.float32)
    coeff = np.asarray(coeff, np.float32)
    _check_tables(raw.shape, dark, coeff)
    g = line_gains(gains)
    keep = keep_bands(wavelengths)
    centers = binned_centers(wavelengths, factor)
    nb = centers.shape[0]
    L, S = raw.shape[:2]
    out = np.empty((L, S, nb), np.float32)
    for lo in range(0, L, chunk_lines):
        hi = min(L, lo + chunk_lines)
        x = raw[lo:hi].astype(np.float32) - dark[None]
        np.maximum(x, np.float32(0.0), out=x)
        x *= coeff[None]
        x /= g[lo:hi, None, None]
        x = x[:, :, keep].reshape(hi - lo, S, nb, factor)
        out[lo:hi] = sequential_sum_f32(x)
    rgb_idx = [band_nearest(centers, t) for t in RGB_TARGETS_NM]
    rgb = np.ascontiguousarray(out[:, :, rgb_idx])
    return out, centers, rgb


# --------------------------------------------------------------------------- statistics
@dataclass(frozen=True)
class Stats:
    """rx.py:26-39 CubeStats, as plain arrays."""

    mu: np.ndarray
    sigma: np.ndarray
    sigma_inv: np.ndarray
    ridge_used: float
    chol_lower: np.ndarray


def factor_covariance(mu, cov) -> Stats:
    """rx.py:68-86 — ridge-escalated Cholesky and the symmetric inverse."""
    bands = cov.shape[0]
    trace = float(np.trace(cov))
    scale = trace / bands if trace > 0 else 1.0
    chol = None
    ridge = 0.0
    for eps in (0.0,) + RIDGE_EPSILONS:
        ridge = eps * scale
        try:
            chol = np.linalg.cholesky(cov + ridge * np.eye(bands))
            break
        except np.linalg.LinAlgError:
            continue
    if chol is None:
        raise ValueError("covariance not positive definite even after ridging")
    inv = cho_solve((chol, True), np.eye(bands), check_finite=False)
    inv = (inv + inv.T) / 2.0
    return Stats(mu=mu, sigma=cov, sigma_inv=inv, ridge_used=ridge, chol_lower=chol)


def compute_stats(values, chunk: int = 65536) -> Stats:
    """rx.py:42-86 — two-pass f64 mean and unbiased covariance over all pixels."""
    values = np.asarray(values, np.float32)
    bands = values.shape[-1]
    px = values.reshape(-1, bands)
    n = px.shape[0]
    if n <= bands:
        raise ValueError(f"insufficient samples: {n} pixels for {bands} bands")
    if not np.isfinite(values).all():
        raise ValueError("invalid data: cube contains non-finite values")
    mu = np.zeros(bands)
    for a in range(0, n, chunk):
        mu += px[a:a + chunk].astype(np.float64).sum(axis=0)
    mu /= n
    cov = np.zeros((bands, bands))
    for a in range(0, n, chunk):
        d = px[a:a + chunk].astype(np.float64) - mu
        cov += d.T @ d
    cov /= n - 1
    cov = (cov + cov.T) / 2.0
    return factor_covariance(mu, cov)


def compute_stats_exact(raw, dark, coeff, gains, chunk_lines: int = 256) -> Stats:
    """rx.py:42-86's algorithm on the EXACT radiance max(raw - dark, 0) * coeff / gain
    (f64 arithmetic, no f32 rounding of the radiance): a diagnostic that splits a
    Sigma^-1 difference into the part the reference's own f32 radiance rounding
    (calibrate.py:98-101) causes and the part a kernel causes.  Two passes over
    line chunks, like rx.py:56-66, so full strips fit in host memory."""
    raw = np.asarray(raw)
    dark = np.asarray(dark, np.float64)
    coeff = np.asarray(coeff, np.float64)
    g = line_gains(gains).astype(np.float64)
    L, S, B = raw.shape
    n = L * S
    if n <= B:
        raise ValueError(f"insufficient samples: {n} pixels for {B} bands")

    def rad(a, b):
        x = np.maximum(raw[a:b].astype(np.float64) - dark[None], 0.0) * coeff[None]
        return (x / g[a:b, None, None]).reshape(-1, B)

    mu = np.zeros(B)
    for a in range(0, L, chunk_lines):
        mu += rad(a, min(L, a + chunk_lines)).sum(axis=0)
    mu /= n
    cov = np.zeros((B, B))
    for a in range(0, L, chunk_lines):
        d = rad(a, min(L, a + chunk_lines)) - mu
        cov += d.T @ d
    cov /= n - 1
    cov = (cov + cov.T) / 2.0
    return factor_covariance(mu, cov)


# --------------------------------------------------------------------------- scoring
def mahalanobis_sq(pixels, mu, chol_lower, chunk: int = 65536) -> np.ndarray:
    """_accel.py:33-47 — delta = ||L^-1 (x - mu)||^2 per row, float64."""
    pixels = np.asarray(pixels)
    n = pixels.shape[0]
    out = np.empty(n)
    for a in range(0, n, chunk):
        d = pixels[a:a + chunk].astype(np.float64) - mu
        y = solve_triangular(chol_lower, d.T, lower=True, check_finite=False)
        out[a:a + chunk] = np.einsum("bn,bn->n", y, y)
    return out


def rx_scores(values, stats: Stats) -> np.ndarray:
    """rx.py:89-97 — f64 scores cast to f32, shaped (lines, samples)."""
    values = np.asarray(values, np.float32)
    if stats.mu.shape[0] != values.shape[-1]:
        raise ValueError(
            f"stats fitted for {stats.mu.shape[0]} bands, cube has {values.shape[-1]}"
        )
    d = mahalanobis_sq(values.reshape(-1, values.shape[-1]), stats.mu, stats.chol_lower)
    return d.reshape(values.shape[:2]).astype(np.float32)


def max_score(scores) -> float:
    """cube.py:174-176."""
    s = np.asarray(scores, np.float32)
    return float(s.max()) if s.size else 0.0


def normalize_scores(scores) -> np.ndarray:
    """rx.py:100-105 — divide by f32(max); unchanged when max <= 0."""
    s = np.asarray(scores, np.float32)
    m = max_score(s)
    if m <= 0.0:
        return s
    return s / np.float32(m)


def threshold_scores(norm_scores, threshold: float) -> np.ndarray:
    """rx.py:108-112 — strict ``>`` compare in f32 (numpy 2 / NEP 50 semantics)."""
    if not 0.0 <= threshold <= 1.0:
        raise ValueError(f"threshold {threshold} outside [0, 1]")
    return np.asarray(norm_scores, np.float32) > np.float32(threshold)


def transmit_domain(values, max_score_: float) -> np.ndarray:
    """rx.py:115-124 — sqrt(v / max) in f64, zeros when max <= 0."""
    v = np.asarray(values, dtype=np.float64)
    if max_score_ <= 0.0:
        return np.zeros_like(v)
    return np.sqrt(np.clip(v / max_score_, 0.0, None))


# --------------------------------------------------------------------------- R-TOPK (new)
def topk_count(n: int, fraction_per_mille: int = 1) -> int:
    """k = ceil(n * 0.001) computed in integers (SURVEY.md §8(a) R-TOPK)."""
    return (n * fraction_per_mille + 999) // 1000


def topk_threshold(scores, k: int | None = None) -> float:
    """The (k+1)-th largest f32 score; -inf when k >= N (everything selected)."""
    s = np.asarray(scores, np.float32).ravel()
    n = s.size
    if k is None:
        k = topk_count(n)
    if k >= n:
        return float("-inf")
    return float(np.partition(s, n - k - 1)[n - k - 1])


def topk_mask(scores, k: int | None = None) -> np.ndarray:
    """R-TOPK: mask = delta > delta_(k+1) (strict, like rx.py:112)."""
    s = np.asarray(scores, np.float32)
    t = topk_threshold(s, k)
    if t == float("-inf"):
        return np.ones(s.shape, bool)
    return s > np.float32(t)


# --------------------------------------------------------------------------- R-GLOBAL / R-STREAM (new)
def moments(values, shift) -> tuple[float, np.ndarray, np.ndarray]:
    """Shifted f64 moments (n, sum(x-c), sum((x-c)(x-c)^T)) of one block."""
    px = np.asarray(values, np.float32).reshape(-1, np.asarray(shift).shape[0])
    d = px.astype(np.float64) - np.asarray(shift, np.float64)
    return float(px.shape[0]), d.sum(axis=0), d.T @ d


def combine_moments(parts):
    """Sum of per-shard moments sharing one shift (the NCCL all-reduce payload)."""
    n = sum(p[0] for p in parts)
    s = sum(p[1] for p in parts)
    q = sum(p[2] for p in parts)
    return n, s, q


def finalize_moments(n, s, q, shift, bands=None) -> Stats:
    """mu = c + s/n; sigma = (Q - s s^T / n) / (n - 1), symmetrised; then rx.py:68-86."""
    shift = np.asarray(shift, np.float64)
    bands = shift.shape[0] if bands is None else bands
    if n <= bands:
        raise ValueError(f"insufficient samples: {n} pixels for {bands} bands")
    mu = shift + s / n
    cov = (q - np.outer(s, s) / n) / (n - 1)
    cov = (cov + cov.T) / 2.0
    return factor_covariance(mu, cov)


class StreamingStats:
    """R-STREAM: exponential-forgetting background, score each chunk after folding it in.

    State (n, s, Q) in f64 around a fixed shift c = f64 mean of chunk 0.
    Update per chunk: n <- lam*n + m, s <- lam*s + sum(x-c), Q <- lam*Q + sum((x-c)(x-c)^T).
    For chunk 0 this is exactly compute_stats(chunk 0) up to rounding.
    """

    def __init__(self, bands: int, forget: float = 0.99):
        self.bands = bands
        self.forget = forget
        self.shift = None
        self.n = 0.0
        self.s = np.zeros(bands)
        self.q = np.zeros((bands, bands))

    def update(self, values) -> Stats:
        px = np.asarray(values, np.float32).reshape(-1, self.bands)
        if not np.isfinite(px).all():
            raise ValueError("invalid data: cube contains non-finite values")
        if self.shift is None:
            self.shift = px.astype(np.float64).mean(axis=0)
        m, s, q = moments(px, self.shift)
        lam = self.forget
        self.n = lam * self.n + m
        self.s = lam * self.s + s
        self.q = lam * self.q + q
        return finalize_moments(self.n, self.s, self.q, self.shift, self.bands)


# --------------------------------------------------------------------------- whole path
def detect(raw, dark, coeff, gains, k: int | None = None):
    """raw -> radiance -> stats -> f32 scores -> top-0.1% mask (one global background)."""
    rad = apply_calibration(raw, dark, coeff, gains)
    stats = compute_stats(rad)
    scores = rx_scores(rad, stats)
    mask = topk_mask(scores, k)
    return stats, scores, mask


# --------------------------------------------------------------------------- link payload
# datalink.py:1-24 (layout), 141-177 (per-pixel encodings), 205-240 (packetize_cube)
PAYLOAD_SAMPLES = 900         # datalink.py:36
HEADER_LEN = 128              # datalink.py:35


def quantize(channel, channel_max: float, levels: int) -> np.ndarray:
    """datalink.py:141-145: round-half-up of x / max * levels in f64, clipped; 0 if max <= 0."""
    if channel_max <= 0.0:
        return np.zeros(np.shape(channel), np.uint16)
    q = np.floor(np.asarray(channel, np.float32).astype(np.float64) / channel_max * levels + 0.5)
    return np.clip(q, 0, levels).astype(np.uint16)


def pack_rgb565(rgb, max_r: float, max_g: float, max_b: float) -> np.ndarray:
    """datalink.py:148-152: R in the high 5 bits, G the middle 6, B the low 5."""
    rgb = np.asarray(rgb)
    return ((quantize(rgb[..., 0], max_r, 31) << 11) | (quantize(rgb[..., 1], max_g, 63) << 5)
            | quantize(rgb[..., 2], max_b, 31)).astype(np.uint16)


def encode_scores_half(scores, max_score: float) -> np.ndarray:
    """datalink.py:163-168: IEEE half of sqrt(score / max) (f64 math), as u16 bits."""
    s = np.asarray(scores, np.float32)
    if max_score <= 0.0:
        return np.zeros(s.shape, np.uint16)
    return np.sqrt(s.astype(np.float64) / max_score).astype(np.float16).view(np.uint16)


def pack_header(cube_id, line_index, lines_per_cube, samples, exposure_start_us, max_score,
                max_r, max_g, max_b, ins_before, ins_after) -> bytes:
    """datalink.py:48-77 + 130-133: the 128-byte little-endian line header."""
    import struct

    head = struct.pack("<4sHHIIIIQffff", b"SKRX", 1, HEADER_LEN, cube_id, line_index,
                       lines_per_cube, samples, exposure_start_us, max_score, max_r, max_g, max_b)
    ins = lambda s: struct.pack("<Qddffff", *s)  # noqa: E731  (ts, lat, lon, alt, roll, pitch, yaw)
    return head + ins(ins_before) + ins(ins_after)


def packetize_cube(cube_id, rgb, scores, line_meta) -> list:
    """datalink.py:205-240: one 3728-byte packet per line; cube maxima in every header.
    ``line_meta``: per line (exposure_start_us, ins_before tuple, ins_after tuple)."""
    rgb = np.asarray(rgb, np.float32)
    scores = np.asarray(scores, np.float32)
    lines = rgb.shape[0]
    max_score = float(scores.max()) if scores.size else 0.0
    mr, mg, mb = (float(rgb[:, :, c].max()) for c in range(3))
    out = []
    for i in range(lines):
        exp, ib, ia = line_meta[i]
        payload = np.empty((rgb.shape[1], 2), "<u2")
        payload[:, 0] = pack_rgb565(rgb[i], mr, mg, mb)
        payload[:, 1] = encode_scores_half(scores[i], max_score)
        out.append(pack_header(cube_id, i, lines, rgb.shape[1], exp, max_score, mr, mg, mb, ib, ia)
                   + payload.tobytes())
    return out


# --------------------------------------------------------------------------- GF(256) erasure code
# fec.py:28-195 and _accel.py:50-70 / 92-107 (gf256_matmul), datalink.py:243-285 (frames)
GF_POLY = 0x11D               # fec.py:28 (generator 2, fec.py:29)
FRAME_HEAD = "<IBBH"          # datalink.py:51: group_id, index, kind, payload length


def gf_tables():
    """fec.py:36-50: antilog table doubled to 510 entries (products need no mod 255), log[0] = 0."""
    exp = np.zeros(510, np.uint8)
    log = np.zeros(256, np.int16)
    v = 1
    for e in range(255):
        exp[e], log[v] = v, e
        v = (v << 1) ^ (GF_POLY if v & 0x80 else 0)
    exp[255:] = exp[:255]
    return log, exp


GF_LOG_T, GF_EXP_T = gf_tables()


def gf_mul(a: int, b: int) -> int:
    return 0 if a == 0 or b == 0 else int(GF_EXP_T[int(GF_LOG_T[a]) + int(GF_LOG_T[b])])


def gf_inv(a: int) -> int:
    if a == 0:
        raise ZeroDivisionError("no inverse of 0 in GF(256)")
    return int(GF_EXP_T[255 - int(GF_LOG_T[a])])


def gf_pow(x: int, n: int) -> int:
    """fec.py:65-70 including its int16 arithmetic: log[x] * n is an int16 product (NEP 50),
    so it wraps for log[x] * n > 32767 (codes with more than ~129 data rows) before the
    floor-mod 255."""
    if n == 0:
        return 1
    if x == 0:
        return 0
    p = (int(GF_LOG_T[x]) * n + 32768) % 65536 - 32768
    return int(GF_EXP_T[p % 255])


def gf256_matmul(mat, data) -> np.ndarray:
    """_accel.py:50-70: out[i] = XOR_j mat[i, j] * data[j] over GF(256) (row-vectorised)."""
    mat = np.asarray(mat, np.uint8)
    data = np.asarray(data, np.uint8)
    out = np.zeros((mat.shape[0], data.shape[1]), np.uint8)
    ld = GF_LOG_T[data].astype(np.int64)
    nz = data != 0
    for j in range(mat.shape[1]):
        for i in np.nonzero(mat[:, j])[0]:
            prod = GF_EXP_T[int(GF_LOG_T[mat[i, j]]) + ld[j]]
            out[i] ^= np.where(nz[j], prod, 0).astype(np.uint8)
    return out


def gf_mat_inv(m) -> np.ndarray:
    """fec.py:82-98: Gauss-Jordan on [m | I]; pivot = first nonzero at or below the diagonal."""
    m = np.asarray(m, np.uint8)
    k = m.shape[0]
    a = np.concatenate([m, np.eye(k, dtype=np.uint8)], axis=1)

    def scaled(row, s):
        return gf256_matmul(np.array([[s]], np.uint8), row[None, :])[0]

    for c in range(k):
        nz = np.nonzero(a[c:, c])[0]
        if nz.size == 0:
            raise np.linalg.LinAlgError("singular matrix over GF(256)")
        p = c + int(nz[0])
        a[[c, p]] = a[[p, c]]
        a[c] = scaled(a[c], gf_inv(int(a[c, c])))
        for r in range(k):
            if r != c and a[r, c]:
                a[r] ^= scaled(a[c], int(a[r, c]))
    return a[:, k:].copy()


def encoding_matrix(k: int, total: int) -> np.ndarray:
    """fec.py:101-115: Vandermonde (total x k) at points 0..total-1, times inv(top k rows)."""
    vand = np.array([[gf_pow(i, j) for j in range(k)] for i in range(total)], np.uint8)
    return gf256_matmul(vand, gf_mat_inv(vand[:k]))


def rs_encode(matrix, k: int, payloads) -> list:
    """fec.py:140-155: parity rows = matrix[k:] @ data over GF(256)."""
    data = np.frombuffer(b"".join(payloads), np.uint8).reshape(k, -1)
    return [row.tobytes() for row in gf256_matmul(np.asarray(matrix)[k:], data)]


def rs_decode(matrix, k: int, received):
    """fec.py:157-195: (data dict, (received, recovered, missing)) from (coded index, bytes)
    pairs; the first k by index are solved against when a data slot is absent."""
    ent = sorted(received, key=lambda e: e[0])
    idx = [i for i, _ in ent]
    if len(set(idx)) != len(idx):
        raise ValueError("duplicate coded index in group")
    out = {i: p for i, p in ent if i < k}
    absent = tuple(i for i in range(k) if i not in out)
    direct = tuple(sorted(out))
    if len(ent) < k or not absent:
        return out, (direct, (), absent)
    use = ent[:k]
    inv = gf_mat_inv(np.asarray(matrix)[[i for i, _ in use]])
    stacked = np.frombuffer(b"".join(p for _, p in use), np.uint8).reshape(k, -1)
    rec = gf256_matmul(inv[list(absent)], stacked)
    for s, row in zip(absent, rec):
        out[s] = row.tobytes()
    return out, (direct, absent, ())


def frames_for_cube(cube_id: int, packets, k: int = 50, parity: int = 25, matrix=None) -> list:
    """datalink.py:243-285: per group of k packets, k data frames then `parity` parity frames;
    group id = cube_id * groups + g; frame = <IBBH header (group, index, kind, length) + payload."""
    import struct

    matrix = encoding_matrix(k, k + parity) if matrix is None else matrix
    groups = len(packets) // k
    out = []
    for g in range(groups):
        chunk = list(packets[g * k:(g + 1) * k])
        gid = cube_id * groups + g
        for i, p in enumerate(chunk):
            out.append(struct.pack(FRAME_HEAD, gid, i, 0, len(p)) + p)
        for i, p in enumerate(rs_encode(matrix, k, chunk)):
            out.append(struct.pack(FRAME_HEAD, gid, k + i, 1, len(p)) + p)
    return out
