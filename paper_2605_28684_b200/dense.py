"""Dense helpers with the reference signatures (``adrom/dense.py``).

``thin_svd`` (dense.py:59-72) runs the one-block Jacobi SVD of the CUDA
library (``adrom_small_svd``) for matrices that fit one thread block's
shared memory (the reduced operators of the online loop).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _dev
from ._lib import Context, ptr
from .errors import DenseError

__all__ = ["SvdResult", "DenseError", "thin_svd", "SVD_CUTOFF", "max_principal_angle"]

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
