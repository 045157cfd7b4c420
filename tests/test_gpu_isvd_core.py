"""The iSVD core SVD (csrc/secular.cuh): K = [[lam Sigma, p], [0, rho]] by the
secular equation of K K^T = diag(d^2) + z z^T, checked against the oracle's
restatement of tracking.py:141-178 (gesdd on K) on the cases that stress a
rank-one-update solver: clustered and repeated singular values (deflation by
rotation), zero coefficients (deflation by z), the degenerate branch, a
snapshot in the span, lambda = 0, and noise-level trailing values."""

import numpy as np
import pytest

from oracle import subspace

pytestmark = pytest.mark.gpu


def _case(n, r, sigma, coef, resid, rng):
    phi = np.linalg.qr(rng.standard_normal((n, r)))[0]
    perp = rng.standard_normal(n)
    perp -= phi @ (phi.T @ perp)
    perp /= np.linalg.norm(perp)
    return phi, np.asarray(sigma, float), phi @ np.asarray(coef, float) + resid * perp


def _check(phi, sigma, y, lam, r, path_ok=(0,)):
    import paper_2605_28684_b200 as P
    got = P.isvd_update(P.ReducedBasis(phi=phi, sigma=sigma), y, lam, r)
    info = P.tracking.last_isvd_info()
    ref_phi, ref_sig, _ = subspace.isvd_update(phi, sigma, y, lam, r)
    gs = np.asarray(got.sigma)
    tol = 1e-12 * ref_sig[0] + 1e-10 * ref_sig
    assert np.all(np.abs(gs - ref_sig) <= tol), np.max(np.abs(gs - ref_sig) / ref_sig)
    # subspaces of well-separated leading values agree (sine-based angle)
    k = int(np.sum(ref_sig > 1e-6 * ref_sig[0]))
    gaps = ref_sig[:k - 1] / ref_sig[1:k] if k > 1 else np.array([])
    cut = k if (k == r or ref_sig[k] < 1e-3 * ref_sig[k - 1]) else 0
    if cut:
        assert subspace.max_angle(ref_phi[:, :cut], np.asarray(got.phi)[:, :cut]) < 1e-9
    assert subspace.orthonormality_defect(np.asarray(got.phi)) < 1e-12
    assert info["core_path"] in path_ok, info
    return info


@pytest.mark.parametrize("r", [16, 64, 128])
def test_core_generic(r):
    rng = np.random.default_rng(r)
    phi, sig, y = _case(4096, r, np.sort(rng.uniform(0.1, 2.0, r))[::-1],
                        rng.standard_normal(r), 0.7, rng)
    _check(phi, sig, y, 0.9, r)


def test_core_repeated_sigma_rotation_deflation():
    rng = np.random.default_rng(1)
    r = 32
    sig = np.repeat([3.0, 1.0, 0.25, 1e-3], 8)
    phi, sig, y = _case(2048, r, sig, rng.standard_normal(r), 0.4, rng)
    _check(phi, sig, y, 0.5, r)


def test_core_zero_coefficients_and_in_span():
    rng = np.random.default_rng(2)
    r = 24
    coef = rng.standard_normal(r)
    coef[::3] = 0.0
    phi, sig, y = _case(2048, r, np.linspace(2.0, 0.5, r), coef, 0.0, rng)
    info = _check(phi, sig, y, 0.8, r)
    assert info["degenerate"]


def test_core_lambda_zero_and_tiny_tail():
    rng = np.random.default_rng(3)
    r = 64
    sig = np.concatenate([[1.0, 1e-3, 1e-6], 1e-12 * (1 + 0.01 * np.arange(r - 3))])
    phi, sig, y = _case(8192, r, sig, 1e-12 * rng.standard_normal(r), 1e-9, rng)
    _check(phi, sig, y, 0.1, r)
    phi, sig, y = _case(8192, r, np.linspace(2, 1, r), rng.standard_normal(r), 0.3, rng)
    _check(phi, sig, y, 0.0, r)


def test_least_squares_far_from_orthonormal_basis():
    """tracking.py:161 (gelsd) on a basis whose Gram matrix is far from the
    identity: the Neumann series of the tracked-Gram solve diverges and the
    block-parallel direct solve (isvd_solve_direct_kernel) takes over."""
    from paper_2605_28684_b200 import ReducedBasis, isvd_update
    from oracle import subspace
    rng = np.random.default_rng(17)
    n, r = 5000, 24
    phi = np.linalg.qr(rng.standard_normal((n, r)))[0]
    phi = phi @ (np.eye(r) + 0.6 * rng.standard_normal((r, r)) / np.sqrt(r))   # G = M^T M, ||G - I|| > 1
    sig = np.linspace(3.0, 0.5, r)
    y = phi @ rng.standard_normal(r) + 0.2 * rng.standard_normal(n)
    got = isvd_update(ReducedBasis(phi, sig), y, 0.7, r)
    ref_phi, ref_sig, _ = subspace.isvd_update(phi, sig, y, 0.7, r)
    assert np.allclose(got.sigma, ref_sig, rtol=1e-9)
    g = np.asarray(got.phi)
    sgn = np.sign(np.sum(g * ref_phi, axis=0))
    rel = np.linalg.norm(g * sgn - ref_phi, axis=0) / np.linalg.norm(ref_phi, axis=0)
    assert rel.max() < 1e-8, rel.max()
