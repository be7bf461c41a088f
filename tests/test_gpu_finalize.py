"""K3 latency kernels (csrc/finalize_panel.cu, B <= 128; finalize_small.cu; finalize_wide.cu,
128 < B <= 288) against the general
finalize_kernel (stats.cu, SKYRX_B200_FIN_GENERAL=1) and the oracle.

Same operands, order and rounding for the factor: mu, sigma, L and W must be
bit-identical to the general kernel, ridge and status equal, for well-posed,
rank-deficient (ridged), non-PD, non-finite and insufficient inputs;
sigma_inv = W^T W is summed in 4 x 4 register tiles (another order), so it is
held to 1e-14 normwise.
"""

import numpy as np
import pytest

from oracle import skyrx_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2602_13509_b200 as P
    from paper_2602_13509_b200 import build

    build.build()
    return P


def moments_batch(B, rng):
    """[n, s, Q] moment blocks about a shift: a spectrum-like well-posed one, a
    rank-deficient one (needs the ridge), a zero one, one with too few pixels."""
    out, shifts = [], []
    for kind in range(4):
        n = 5000 if kind != 3 else B
        basis = rng.standard_normal((max(1, B // 3), B))
        if kind == 0:
            X = rng.standard_normal((n, B)) @ np.diag(np.linspace(1, 30, B)) + 50
        elif kind == 1:
            X = rng.standard_normal((n, basis.shape[0])) @ basis + 7
        elif kind == 2:
            X = np.full((n, B), 3.0)
        else:
            X = rng.standard_normal((n, B))
        c = X[:64].mean(0)
        d = X - c
        out.append(np.concatenate([[float(n)], d.sum(0), (d.T @ d).ravel()]))
        shifts.append(c)
    return np.stack(out), np.stack(shifts)


def finalize(P, mom, shift, B, monkeypatch, general):
    import torch
    from paper_2602_13509_b200 import _dev, _lib

    if general:
        monkeypatch.setenv("SKYRX_B200_FIN_GENERAL", "1")
    else:
        monkeypatch.delenv("SKYRX_B200_FIN_GENERAL", raising=False)
    ds = P.DeviceStats(B, batch=mom.shape[0])
    ds.moments.copy_(torch.from_numpy(mom))
    ds.shift.copy_(torch.from_numpy(shift))
    ds.finalize()
    torch.cuda.synchronize()
    return {k: getattr(ds, k).cpu().numpy() for k in
            ("mu", "sigma", "chol", "sigma_inv", "w64", "whiten", "mu_hilo", "ridge", "status")}


@pytest.mark.parametrize("B", [1, 3, 16, 31, 32, 33, 44, 45, 63, 70, 79, 80, 96, 97, 119, 128,
                               129, 160, 161, 200, 255, 270, 272, 288])
def test_small_equals_general(P, monkeypatch, B):
    rng = np.random.default_rng(B)
    mom, shift = moments_batch(B, rng)
    a = finalize(P, mom, shift, B, monkeypatch, general=False)
    b = finalize(P, mom, shift, B, monkeypatch, general=True)
    assert np.array_equal(a["status"], b["status"])
    assert np.array_equal(a["ridge"], b["ridge"])
    ok = a["status"] == 0
    # B > 118: the general path takes W from its column-wise multi-CTA kernel (another
    # summation order; finalize_wide.cu: a blocked one), so W and its f32 copy are compared
    # to rounding there
    exact = ("mu", "sigma", "chol") + (("w64", "whiten", "mu_hilo") if B <= 118 else ("mu_hilo",))
    for key in exact:
        for m in np.flatnonzero(ok):
            assert np.array_equal(a[key][m].view(np.uint8), b[key][m].view(np.uint8)), (key, m)
    # two backward-stable triangular inverses agree to rounding x cond(L); the ridged
    # rank-deficient matrix (m = 1, cond(L) ~ 1e5) widens that for the blocked wide kernel
    tol = 1e-13 if B <= 128 else 1e-11
    if B > 118:
        for m in np.flatnonzero(ok):
            d = np.abs(a["w64"][m] - b["w64"][m]).max()
            assert d <= tol * np.abs(b["w64"][m]).max(), (m, d)
    for m in np.flatnonzero(ok):
        d = np.abs(a["sigma_inv"][m] - b["sigma_inv"][m]).max()
        assert d <= tol / 10 * np.abs(b["sigma_inv"][m]).max(), (m, d)
        assert np.array_equal(a["sigma_inv"][m], a["sigma_inv"][m].T)
    # and the oracle's factorisation of the same moments (rx.py:56-86); the ridged
    # rank-deficient case (cond ~ 1e10) only on its ridge
    for m in np.flatnonzero(ok):
        if m == 1:
            want = O.finalize_moments(mom[m, 0], mom[m, 1:1 + B], mom[m, 1 + B:].reshape(B, B),
                                      shift[m], B)
            assert a["ridge"][m] == pytest.approx(want.ridge_used, rel=1e-14)
            continue
        B_ = B
        want = O.finalize_moments(mom[m, 0], mom[m, 1:1 + B_], mom[m, 1 + B_:].reshape(B_, B_),
                                  shift[m], B_)
        assert a["ridge"][m] == pytest.approx(want.ridge_used, rel=1e-14)
        assert np.allclose(a["chol"][m], want.chol_lower, rtol=1e-9, atol=1e-12 *
                           np.abs(want.chol_lower).max())
        err = np.abs(a["sigma_inv"][m] - want.sigma_inv).max() / np.abs(want.sigma_inv).max()
        assert err < 1e-8, (m, err)
    assert a["status"][3] != 0   # insufficient samples


def test_nonfinite_and_range_flags(P):
    import torch

    B = 70
    rng = np.random.default_rng(3)
    mom, shift = moments_batch(B, rng)
    ds = P.DeviceStats(B, batch=4)
    ds.moments.copy_(torch.from_numpy(mom))
    ds.shift.copy_(torch.from_numpy(shift))
    ds.flags.copy_(torch.tensor([1, 4, 2, 0], dtype=torch.int32))
    ds.finalize()
    st = ds.status.cpu().numpy()
    from paper_2602_13509_b200 import _lib

    assert st[0] == _lib.ERR_NONFINITE and st[1] == _lib.ERR_RANGE and st[2] == _lib.ERR_RANGE


@pytest.mark.parametrize("B", [16, 45, 70, 80])
def test_panel_equals_slot(P, monkeypatch, B):
    """The panel kernel and the per-column slot kernel: bit-identical outputs."""
    rng = np.random.default_rng(100 + B)
    mom, shift = moments_batch(B, rng)
    a = finalize(P, mom, shift, B, monkeypatch, general=False)
    monkeypatch.setenv("SKYRX_B200_FIN_SLOT", "1")
    b = finalize(P, mom, shift, B, monkeypatch, general=False)
    monkeypatch.delenv("SKYRX_B200_FIN_SLOT", raising=False)
    for key in ("status", "ridge", "mu", "sigma", "chol", "w64", "whiten", "mu_hilo", "sigma_inv"):
        for m in range(mom.shape[0]):
            if key not in ("status", "ridge") and a["status"][m] != 0:
                continue
            assert np.array_equal(np.atleast_1d(a[key][m]).view(np.uint8),
                                  np.atleast_1d(b[key][m]).view(np.uint8)), (key, m)
