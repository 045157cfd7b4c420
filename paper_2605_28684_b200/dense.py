"""Dense helpers with the reference signatures (``adrom/dense.py``).

``thin_svd`` (dense.py:59-72) runs the one-block Jacobi SVD of the CUDA
library (``adrom_small_svd``) for matrices that fit one thread block's
shared memory (the reduced operators of the online loop).  ``orth``,
``least_squares`` (Householder QR + one-sided Jacobi, csrc/hhqr.cu /
offline.cu), ``pivoted_qr`` (the exact-greedy QDEIM kernel for the pivots),
``principal_angles`` and ``newton_solve`` (callbacks on the host, the
dense LU solve on the device) complete the reference module.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _dev
from ._lib import Context, ptr
from .errors import DenseError

__all__ = ["SvdResult", "NewtonResult", "DenseError", "thin_svd", "pivoted_qr", "least_squares",
           "principal_angles", "newton_solve", "orth", "fix_column_signs", "pinv_cut",
           "SVD_CUTOFF", "max_principal_angle"]

SVD_CUTOFF = 1e-12  # dense.py:32


@dataclass(frozen=True)
class SvdResult:
    """dense.py:46-56."""

    u: object
    s: object
    v: object


def thin_svd(a) -> SvdResult:
    """dense.py:59-72 — economy SVD, singular values descending."""
    ad = _dev.dev(a)
    if ad.dim() != 2 or ad.shape[0] < 1 or ad.shape[1] < 1:
        raise DenseError(f"thin_svd expects a non-empty 2-d array, got shape {tuple(ad.shape)}")
    m, n = ad.shape
    k = min(m, n)
    u = _dev.empty(m, k)
    s = _dev.empty(k)
    v = _dev.empty(n, k)
    Context.get().call("adrom_small_svd", ptr(ad), C.c_int32(m), C.c_int32(n), ptr(u), ptr(s),
                       ptr(v))
    return SvdResult(u=_dev.like(u, a), s=_dev.like(s, a), v=_dev.like(v, a))


def max_principal_angle(u, v) -> float:
    """Largest principal angle between two orthonormal spans via the explicit
    residual R = V - U (U^T V) (sine-based, SURVEY §8c convention 2); works
    on device tensors of any height."""
    t = _dev.torch()
    ud, vd = _dev.dev(u), _dev.dev(v)
    resid = vd - ud @ (ud.T @ vd)
    smax = float(t.linalg.svdvals(resid.T @ resid).max().sqrt()) if resid.numel() else 0.0
    return float(np.arcsin(min(smax, 1.0)))


def ts_tn(a, b, a_kmajor: bool = False):
    """A^T B for tall A (K x m, or m x K when ``a_kmajor``) and B (K x n) on the
    FP64 tensor cores (``adrom_ts_tn``, deterministic split-K); m <= 128,
    n <= 136.  Device tensors in, device (m x n) tensor out."""
    t = _dev.torch()
    ad, bd = _dev.dev(a).contiguous(), _dev.dev(b).contiguous()
    m = ad.shape[0] if a_kmajor else ad.shape[1]
    k = ad.shape[1] if a_kmajor else ad.shape[0]
    if bd.shape[0] != k:
        raise ValueError(f"inner dimensions differ: {tuple(ad.shape)} vs {tuple(bd.shape)}")
    n = bd.shape[1]
    c = t.empty((n, m), dtype=t.float64, device="cuda")  # column-major m x n
    Context.get().call("adrom_ts_tn", C.c_int64(k), C.c_int32(m), C.c_int32(n), ptr(ad),
                       C.c_int64(ad.shape[1]), C.c_int32(1 if a_kmajor else 0), ptr(bd),
                       C.c_int64(n), ptr(c))
    return c.T


def ts_apply(a, m_mat, out_kmajor: bool = False):
    """A M for tall A (K x m) and small M (m x n) on the FP64 tensor cores
    (``adrom_ts_apply``); returns K x n (or its n x K transpose storage when
    ``out_kmajor``, as an n x K tensor)."""
    t = _dev.torch()
    ad, md = _dev.dev(a).contiguous(), _dev.dev(m_mat).contiguous()
    k, m = ad.shape
    if md.shape[0] != m:
        raise ValueError(f"inner dimensions differ: {tuple(ad.shape)} vs {tuple(md.shape)}")
    n = md.shape[1]
    out = t.empty((n, k) if out_kmajor else (k, n), dtype=t.float64, device="cuda")
    Context.get().call("adrom_ts_apply", C.c_int64(k), C.c_int32(m), C.c_int32(n), ptr(ad),
                       C.c_int64(m), ptr(md), ptr(out), C.c_int64(k if out_kmajor else n),
                       C.c_int32(1 if out_kmajor else 0))
    return out


def least_squares(a, b):
    """dense.py:100-111 — minimizer of ||a x - b|| for a tall ``a`` (minimum
    norm, singular values below 1e-12 s_max discarded, as gelsd)."""
    ad = _dev.dev(a)
    bd = _dev.dev(b)
    if ad.dim() != 2:
        raise DenseError(f"least_squares expects a 2-d matrix, got shape {tuple(ad.shape)}")
    n, k = ad.shape
    if n < k:
        raise DenseError(f"least_squares expects rows >= cols, got shape {tuple(ad.shape)}")
    vec = bd.dim() == 1
    b2 = bd.reshape(n, -1).contiguous()
    if b2.shape[0] != n:
        raise ValueError(f"rhs rows {b2.shape[0]} do not match matrix rows {n}")
    x = _dev.empty(k, b2.shape[1])
    Context.get().call("adrom_least_squares", ptr(ad), C.c_int64(n), C.c_int32(k), ptr(b2),
                       C.c_int32(b2.shape[1]), ptr(x))
    x = x.reshape(k) if vec else x
    return _dev.like(x, a)


def orth(a):
    """dense.py:175-179 — thin-QR orthonormalisation, largest-|.| entry of
    each column made nonnegative."""
    ad = _dev.dev(a)
    n, m = ad.shape
    if n < m:
        raise DenseError(f"orth expects a tall matrix, got shape {tuple(ad.shape)}")
    q = _dev.empty(n, m)
    Context.get().call("adrom_orth", ptr(ad), C.c_int64(n), C.c_int32(m), ptr(q))
    return _dev.like(q, a)


def fix_column_signs(q):
    """dense.py:182-189 (device reduction per column via torch's first-index
    argmax, then a sign flip)."""
    t = _dev.torch()
    qd = _dev.dev(q)
    lead = qd.abs().argmax(dim=0)
    signs = t.sign(qd[lead, t.arange(qd.shape[1], device=qd.device)])
    signs = t.where(signs == 0, t.ones_like(signs), signs)
    return _dev.like(qd * signs, q)


def pinv_cut(a):
    """dense.py:192-200 — pseudo-inverse with the 1e-12 relative cutoff."""
    t = _dev.torch()
    res = thin_svd(_dev.dev(a))
    s = res.s
    smax = s[0] if s.numel() else t.zeros((), dtype=s.dtype, device=s.device)
    keep = s > SVD_CUTOFF * smax
    inv = t.where(keep, 1.0 / t.where(keep, s, t.ones_like(s)), t.zeros_like(s))
    out = ts_apply((res.v * inv).contiguous(), res.u.T.contiguous())
    return _dev.like(out, a)


def pivoted_qr(a, k: int):
    """dense.py:75-97 — greedy column-pivoted QR, first ``k`` pivots.

    The pivots are the exact-greedy selection of the QDEIM kernel (the column
    of largest residual norm at each step, ties to the lowest index); the
    remaining columns follow in index order, and (q, r) is the Householder QR
    of the permuted matrix, so ``a[:, piv] = q r``."""
    t = _dev.torch()
    ad = _dev.dev(a)
    if not bool(t.isfinite(ad).all()):
        raise DenseError("pivoted_qr input contains non-finite entries")
    m, n = ad.shape
    if k > n:
        raise DenseError(f"requested {k} pivots from a matrix with {n} columns")
    kk = min(m, n)
    if k > kk:
        raise DenseError(f"pivoted_qr: matrix has at most rank {kk}, cannot select {k} pivots")
    idx = _dev.empty(kk, dtype=t.int64)
    at = ad.T.contiguous()
    Context.get().call("adrom_qdeim", ptr(at), C.c_int64(n), C.c_int32(m),
                       C.c_int32(kk), ptr(idx))
    rest = t.ones(n, dtype=t.bool, device="cuda")
    rest[idx] = False
    piv = t.cat([idx, t.arange(n, device="cuda")[rest]])
    ap = ad[:, piv]
    q = orth(ap[:, :kk])
    r = t.triu(ts_tn(q, ap))
    rdiag = r.diagonal().abs()
    for j in range(min(k, kk)):
        if float(rdiag[j]) < 1e-14:
            raise DenseError(f"pivoted_qr: rank deficient at pivot step {j} "
                             f"(residual column norm {float(rdiag[j]):.3e})")
    return (_dev.like(piv[:k].clone(), a), _dev.like(q, a), _dev.like(r, a))


def principal_angles(u, v):
    """dense.py:114-126 — canonical angles (ascending), small angles by the
    sine branch (scipy.linalg.subspace_angles' recipe) with the residual
    V - U (U^T V) formed on the tensor cores."""
    t = _dev.torch()
    ud, vd = _dev.dev(u), _dev.dev(v)
    if ud.shape[0] != vd.shape[0]:
        raise DenseError(f"row mismatch: {tuple(ud.shape)} vs {tuple(vd.shape)}")
    if ud.shape[1] < vd.shape[1]:
        ud, vd = vd, ud
    qa, qb = orth(ud), orth(vd)
    c = ts_tn(qa, qb)
    sig = thin_svd(c).s.clamp(max=1.0)
    resid = qb - ts_apply(qa, c)
    sb = thin_svd(ts_tn(resid, resid)).s.clamp(min=0.0).sqrt().clamp(max=1.0).flip(0)
    mask = sig * sig >= 0.5
    theta = t.where(mask, t.arcsin(sb), t.arccos(sig))
    return _dev.like(t.sort(theta).values, u)


@dataclass
class NewtonResult:
    """dense.py:129-137."""

    x: object
    converged: bool
    iterations: int
    residual_norm: float


def newton_solve(residual, jacobian, x0, tol: float, max_iter: int) -> NewtonResult:
    """dense.py:140-171 — dense Newton; each step solves J d = -r by LU with
    partial pivoting on the device (adrom_lu_solve).  ``residual`` /
    ``jacobian`` are user callbacks (numpy or device tensors)."""
    t = _dev.torch()
    if tol <= 0:
        raise DenseError("newton_solve requires tol > 0")
    x = _dev.dev(x0).clone()

    def _finite(name, arr):
        a = _dev.dev(arr)
        if not bool(t.isfinite(a).all()):
            raise DenseError(f"{name} contains non-finite entries")
        return a

    back = (lambda z: _dev.like(z, x0))
    r = _finite("newton residual", residual(back(x)))
    rnorm = float(t.linalg.vector_norm(r))
    for it in range(max_iter):
        if rnorm <= tol:
            return NewtonResult(x=back(x), converged=True, iterations=it, residual_norm=rnorm)
        jac = _finite("newton jacobian", jacobian(back(x))).contiguous()
        n = x.shape[0]
        d = (-r).contiguous()
        try:
            Context.get().call("adrom_lu_solve", ptr(jac), C.c_int64(n), ptr(d))
        except DenseError as exc:
            raise DenseError(f"singular Jacobian at Newton iteration {it}") from exc
        x = x + d
        r = _finite("newton residual", residual(back(x)))
        rnorm = float(t.linalg.vector_norm(r))
    return NewtonResult(x=back(x), converged=rnorm <= tol, iterations=max_iter, residual_norm=rnorm)
