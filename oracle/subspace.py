"""Oracle: thin SVD, incremental SVD update, subspace comparison.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Restates ``/root/reference/pkg/src/adrom/tracking.py:141-178`` (``isvd_update``)
and the dense helpers it uses from ``dense.py`` (``thin_svd`` 59-72,
``least_squares`` 100-111, ``principal_angles`` 114-126).  The numerical
kernels are the same LAPACK drivers the reference calls (gesdd, gelsd), so
on identical inputs the oracle reproduces the reference bit for bit on the
same machine; ``tests/golden`` pins that.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg

from .physics import OracleDenseError

#: relative singular value cutoff of every pseudo-inverse (dense.py:32)
SVD_CUTOFF = 1e-12
#: relative residual threshold of the degenerate iSVD branch (tracking.py:46)
DEGENERATE_TOL = 1e-12


def _finite(name, a):
    """dense.py:39-43."""
    a = np.asarray(a, dtype=float)
    if not np.all(np.isfinite(a)):
        raise OracleDenseError(f"{name} contains non-finite entries")
    return a


def thin_svd(a):
    """dense.py:59-72 — economy SVD (gesdd), values descending.

    Returns (u, s, v) with v = vt.T.
    """
    a = _finite("thin_svd input", a)
    if a.ndim != 2 or min(a.shape) < 1:
        raise OracleDenseError(f"thin_svd expects a non-empty 2-d array, got {a.shape}")
    try:
        u, s, vt = np.linalg.svd(a, full_matrices=False)
    except np.linalg.LinAlgError as exc:
        raise OracleDenseError(f"SVD did not converge: {exc}") from exc
    return u, s, vt.T


def lstsq(a, b):
    """dense.py:100-111 — gelsd with rcond = SVD_CUTOFF."""
    a = _finite("least_squares matrix", a)
    b = _finite("least_squares rhs", b)
    if a.shape[0] < a.shape[1]:
        raise OracleDenseError(f"least_squares expects rows >= cols, got {a.shape}")
    return np.linalg.lstsq(a, b, rcond=SVD_CUTOFF)[0]


def core_matrix(sigma, p, qnorm, ynorm, lam):
    """tracking.py:166-173 — K = [[lam*Sigma, p], [0, ||q||]]; the last row
    stays zero when ||q|| <= 1e-12 * max(||y||, 1e-300)."""
    r_cur = sigma.size
    k = np.zeros((r_cur + 1, r_cur + 1))
    k[:r_cur, :r_cur] = np.diag(lam * sigma)
    k[:r_cur, r_cur] = p
    degenerate = qnorm <= DEGENERATE_TOL * max(ynorm, 1e-300)
    if not degenerate:
        k[r_cur, r_cur] = qnorm
    return k, degenerate


def isvd_update(phi, sigma, y_hat, lam, r, projection="lstsq"):
    """tracking.py:141-178 — rank-r Brand update with forgetting ``lam``.

    ``projection="lstsq"`` is the reference's p = Phi^+ y (gelsd);
    ``"gram"`` uses p = Phi^T y (valid for orthonormal Phi; used only to
    time the oracle at sizes where gelsd of an N x r matrix is too slow).
    Returns (phi_new, sigma_new, info) with info = dict(p, qnorm, ynorm,
    degenerate, core_u, core_s).
    """
    y_hat = np.asarray(y_hat, dtype=float)
    n, r_cur = phi.shape
    if y_hat.shape != (n,):
        raise ValueError(f"snapshot length {y_hat.shape} does not match basis rows {n}")
    if projection == "lstsq":
        p = lstsq(phi, y_hat)
    else:
        p = _finite("least_squares matrix", phi).T @ _finite("least_squares rhs", y_hat)
    q = y_hat - phi @ p
    qnorm = float(np.linalg.norm(q))
    ynorm = float(np.linalg.norm(y_hat))
    k, degenerate = core_matrix(np.asarray(sigma, dtype=float), p, qnorm, ynorm, lam)
    q_unit = np.zeros(n) if degenerate else q / qnorm
    u, s, _ = thin_svd(k)
    phi_new = np.column_stack([phi, q_unit]) @ u[:, :r]
    info = dict(p=p, qnorm=qnorm, ynorm=ynorm, degenerate=degenerate, core_u=u, core_s=s)
    return phi_new, s[:r].copy(), info


def principal_angles(u, v):
    """dense.py:114-126 — sine-safe canonical angles, ascending."""
    u = _finite("principal_angles U", u)
    v = _finite("principal_angles V", v)
    if u.shape[0] != v.shape[0]:
        raise OracleDenseError(f"row mismatch: {u.shape} vs {v.shape}")
    return np.sort(scipy.linalg.subspace_angles(u, v))


def max_angle(u, v):
    """Largest principal angle between two orthonormal column spans via the
    explicit residual R = V - U (U^T V): sin(theta_max) = sigma_max(R).

    Equivalent to ``principal_angles(u, v).max()`` for small angles (SURVEY
    §8c convention 2) but costs two tall-skinny products instead of an
    N x r SVD, so it can run at N = 2^24.
    """
    u = np.asarray(u, dtype=float)
    v = np.asarray(v, dtype=float)
    resid = v - u @ (u.T @ v)
    gram = resid.T @ resid
    smax = np.sqrt(max(float(np.linalg.eigvalsh(gram).max()), 0.0))
    return float(np.arcsin(min(smax, 1.0)))


def orthonormality_defect(phi):
    """tracking.py:62-64 — ||Phi^T Phi - I||_F."""
    r = phi.shape[1]
    return float(np.linalg.norm(phi.T @ phi - np.eye(r)))


def fix_column_signs(q):
    """dense.py:182-189 — largest-magnitude entry of each column >= 0."""
    q = np.array(q, dtype=float)
    lead = np.abs(q).argmax(axis=0)
    signs = np.sign(q[lead, np.arange(q.shape[1])])
    signs[signs == 0] = 1.0
    return q * signs


def pod(snapshots, r):
    """snapshots.py:72-89 — leading r left singular vectors of the
    preprocessed snapshot matrix, sign-fixed, with the numerical-rank check."""
    snapshots = np.asarray(snapshots, dtype=float)
    if r > min(snapshots.shape):
        raise OracleDenseError(f"cannot extract {r} modes from {snapshots.shape}")
    u, s, _ = thin_svd(snapshots)
    rank = int(np.sum(s > 1e-12 * s[0])) if s[0] > 0 else 0
    if r > rank:
        raise OracleDenseError(f"requested {r} modes but snapshot matrix has numerical rank {rank}")
    return fix_column_signs(u[:, :r]), s[:r].copy()


def fit_scaling(training, n_var):
    """snapshots.py:54-69 (+ driver.py:232-247 unit branch for n_var == 1).

    Returns (q_ref, phi_norm)."""
    q_ref = np.asarray(training[0], dtype=float).copy()
    if n_var == 1:
        return q_ref, np.ones(1)
    fluct = np.stack([np.asarray(q, dtype=float) - q_ref for q in training])
    per_var = fluct.reshape(len(training), -1, n_var) ** 2
    phi_norm = np.maximum(per_var.mean(axis=(0, 1)), 1e-30)
    phi_norm[phi_norm <= 1e-30] = 1.0
    return q_ref, phi_norm


def row_scale(phi_norm, n_elem):
    """snapshots.py:42-45 — tile(1/phi_norm, n_elem)."""
    return np.tile(1.0 / np.asarray(phi_norm, dtype=float), n_elem)
