"""Device-resident basis tracking: ``ReducedBasis`` and the iSVD update.

Mirrors ``/root/reference/pkg/src/adrom/tracking.py``: ``ReducedBasis``
(51-64), ``SnapshotWindow`` (67-93), ``UpdateRule`` (96-138),
``isvd_update`` (141-178) and the other five rules (181-246: wsvd, direct,
onestep, oja, grouse).  The iSVD is the north-star path
(its own fused kernels); the other rules are host-orchestrated chains of the
library's dense kernels (Householder QR / orth, least squares, one-sided
Jacobi SVD, FP64 tensor-core tall-skinny products).
"""

from __future__ import annotations

import ctypes as C
from collections import deque
from dataclasses import dataclass

import numpy as np

from . import _dev
from ._lib import Context, IsvdInfo, ptr

__all__ = ["ReducedBasis", "SnapshotWindow", "UpdateRule", "isvd_update", "wsvd_update",
           "direct_update", "onestep_update", "oja_update", "grouse_update", "DEGENERATE_TOL",
           "SKIP_TOL", "last_isvd_info"]

DEGENERATE_TOL = 1e-12  # tracking.py:46
SKIP_TOL = 1e-14        # tracking.py:48


@dataclass(frozen=True)
class ReducedBasis:
    """tracking.py:51-64 — orthonormal basis (N x r) + singular values."""

    phi: object
    sigma: object

    @property
    def rank(self) -> int:
        return int(self.phi.shape[1])

    def orthonormality_defect(self) -> float:
        if _dev.is_device(self.phi):
            t = _dev.torch()
            g = self.phi.T @ self.phi
            return float(t.linalg.norm(g - t.eye(self.rank, dtype=g.dtype, device=g.device)))
        r = self.rank
        return float(np.linalg.norm(self.phi.T @ self.phi - np.eye(r)))


class SnapshotWindow:
    """tracking.py:67-93 — ring buffer of the most recent preprocessed
    snapshots (device vectors), initialised from the last
    ``min(capacity, available)`` offline snapshots."""

    def __init__(self, capacity: int, initial=None):
        if capacity < 1:
            raise ValueError("window capacity must be at least 1")
        self.capacity = int(capacity)
        self._buf: deque = deque(maxlen=self.capacity)
        init = list(initial) if initial is not None else []
        for y in init[-self.capacity:]:
            self._buf.append(_dev.dev(y).clone())

    def push(self, y_hat) -> None:
        self._buf.append(_dev.dev(y_hat).clone())

    def __len__(self) -> int:
        return len(self._buf)

    @property
    def matrix(self):
        """N x len column matrix (device)."""
        if not self._buf:
            raise ValueError("snapshot window is empty")
        return _dev.torch().stack(list(self._buf), dim=1).contiguous()


@dataclass(frozen=True)
class UpdateRule:
    """tracking.py:96-138."""

    kind: str
    lam: float = 1.0
    window: int = 8
    eta: float = 0.01

    HISTORY_AWARE = ("isvd", "wsvd", "direct")
    INSTANTANEOUS = ("onestep", "oja", "grouse")

    def __post_init__(self):
        if self.kind not in self.HISTORY_AWARE + self.INSTANTANEOUS:
            raise ValueError(f"unknown update rule {self.kind!r}")
        if not 0.0 <= self.lam <= 1.0:
            raise ValueError("forgetting factor must lie in [0, 1]")
        if self.eta <= 0.0:
            raise ValueError("learning rate must be positive")
        if self.window < 1:
            raise ValueError("window size must be at least 1")

    @property
    def history_aware(self) -> bool:
        return self.kind in self.HISTORY_AWARE

    @property
    def uses_window(self) -> bool:
        return self.kind in ("wsvd", "direct")

    def label(self) -> str:
        if self.kind == "isvd":
            return f"isvd(lambda={self.lam:g})"
        if self.kind in ("wsvd", "direct"):
            return f"{self.kind}(w={self.window})"
        if self.kind == "onestep":
            return "onestep"
        return f"{self.kind}(eta={self.eta:g})"


_last_info = {}


def last_isvd_info() -> dict:
    """Diagnostics of the most recent ``isvd_update`` call (qnorm, ynorm,
    proj_resid, degenerate, reorthogonalised, sweeps, core_path: 0 = secular
    equation, 1/2 = Jacobi fallbacks)."""
    return dict(_last_info)


def isvd_update(basis: ReducedBasis, y_hat, lam: float, r: int) -> ReducedBasis:
    """tracking.py:141-178 — rank-r incremental SVD with forgetting ``lam``.

    Runs three device passes (projection, optional re-orthogonalisation,
    fused rotation) around a one-block SVD of the (r+1)^2 core matrix
    (secular equation of the arrow structure; Jacobi as the verified fallback).  Returns a new basis (inputs are not modified), on the device
    if the inputs were device tensors, else as numpy arrays.
    """
    phi = _dev.dev(basis.phi)
    n, r_cur = phi.shape
    y = _dev.dev(y_hat)
    if y.dim() != 1 or y.shape[0] != n:
        raise ValueError(f"snapshot length {tuple(y.shape)} does not match basis rows {n}")
    sigma = _dev.dev(basis.sigma)
    phi_out = _dev.empty(n, r)
    sigma_out = _dev.empty(r)
    info = IsvdInfo()
    Context.get().call("adrom_isvd_update", ptr(phi), ptr(sigma), ptr(y), C.c_int64(n),
                       C.c_int32(r_cur), C.c_int32(r), C.c_double(lam), ptr(phi_out),
                       ptr(sigma_out), None, C.byref(info))
    _last_info.update(qnorm=info.qnorm, ynorm=info.ynorm, proj_resid=info.proj_resid,
                      degenerate=bool(info.degenerate),
                      reorthogonalised=bool(info.reorthogonalised), sweeps=info.sweeps,
                      core_path=info.core_path)
    return ReducedBasis(phi=_dev.like(phi_out, basis.phi), sigma=_dev.like(sigma_out, basis.sigma))


def wsvd_update(window: SnapshotWindow, r: int) -> ReducedBasis:
    """tracking.py:181-186 — POD of the current window."""
    from .snapshots import pod
    return pod(window.matrix, r)


def direct_update(basis: ReducedBasis, window: SnapshotWindow) -> ReducedBasis:
    """tracking.py:189-203 — Phi' = Y (Phi^+ Y)^+, orthonormalised."""
    from .dense import least_squares, pinv_cut, ts_apply, orth
    from .errors import DenseError
    t = _dev.torch()
    y = window.matrix
    phi = _dev.dev(basis.phi)
    r = phi.shape[1]
    if y.shape[1] < r:
        raise DenseError(f"direct update needs at least {r} window columns, have {y.shape[1]}")
    z = least_squares(phi, y)                     # r x w
    phi_tilde = ts_apply(y, pinv_cut(z))          # N x r
    q = orth(phi_tilde)
    rdiag = ts_tn_diag(q, phi_tilde).abs()        # |diag(R)| of phi_tilde = Q R
    if float(rdiag.min()) <= 1e-12 * max(float(rdiag.max()), 1e-300):
        raise DenseError("direct update produced a rank-deficient basis")
    return ReducedBasis(phi=_dev.like(q, basis.phi), sigma=_dev.like(_dev.dev(basis.sigma).clone(), basis.sigma))


def ts_tn_diag(q, a):
    """diag(Q^T A) on the tensor cores (the R diagonal of A = Q R)."""
    from .dense import ts_tn
    return ts_tn(q, a).diagonal()


def onestep_update(basis: ReducedBasis, y_prev_hat, a_minus) -> ReducedBasis:
    """tracking.py:206-216 — rank-one correction of the projection error of
    the latest snapshot at the predicted reduced state (skipped when the
    reduced state is numerically zero)."""
    from .dense import orth, ts_apply
    t = _dev.torch()
    a = _dev.dev(a_minus)
    denom = float(t.dot(a, a))
    if denom < SKIP_TOL ** 2:
        return basis
    phi = _dev.dev(basis.phi)
    resid = _dev.dev(y_prev_hat) - ts_apply(phi, a[:, None]).reshape(-1)
    phi_new = orth(phi + t.outer(resid, a) / denom)
    return ReducedBasis(phi=_dev.like(phi_new, basis.phi), sigma=_dev.like(_dev.dev(basis.sigma).clone(), basis.sigma))


def oja_update(basis: ReducedBasis, y_prev_hat, eta: float) -> ReducedBasis:
    """tracking.py:219-224 — Oja step + orthonormalisation."""
    from .dense import orth, ts_tn
    t = _dev.torch()
    y = _dev.dev(y_prev_hat)
    phi = _dev.dev(basis.phi)
    yp = ts_tn(y[:, None], phi).reshape(-1)      # y^T Phi
    phi_new = orth(phi + eta * t.outer(y, yp))
    return ReducedBasis(phi=_dev.like(phi_new, basis.phi), sigma=_dev.like(_dev.dev(basis.sigma).clone(), basis.sigma))


def grouse_update(basis: ReducedBasis, y_prev_hat, eta: float) -> ReducedBasis:
    """tracking.py:227-246 — rank-one Grassmannian geodesic step (skipped
    when the snapshot has no in-span part, no residual or zero weights)."""
    import math
    from .dense import least_squares, ts_apply
    t = _dev.torch()
    y = _dev.dev(y_prev_hat)
    phi = _dev.dev(basis.phi)
    w = least_squares(phi, y)
    p = ts_apply(phi, w[:, None]).reshape(-1)
    resid = y - p
    pnorm = float(t.linalg.vector_norm(p))
    rnorm = float(t.linalg.vector_norm(resid))
    wnorm = float(t.linalg.vector_norm(w))
    if min(pnorm, rnorm, wnorm) < SKIP_TOL:
        return basis
    alpha = eta * pnorm * rnorm
    step = (math.cos(alpha) - 1.0) * p / pnorm + math.sin(alpha) * resid / rnorm
    phi_new = phi + t.outer(step, w / wnorm)
    return ReducedBasis(phi=_dev.like(phi_new, basis.phi), sigma=_dev.like(_dev.dev(basis.sigma).clone(), basis.sigma))


class IsvdStream:
    """Streaming form of ``isvd_update`` (B200 extension, r in {32, 64}).

    Repeated ``basis = isvd_update(basis, y, lam, r)`` rewrites the N x r
    basis every update (the O(N r^2) rotation, tracking.py:176-177).  The
    stream keeps the same sequence of bases factored on the device,
    Phi = [A | Q] W (csrc/factored.cu): an update costs two passes over the
    basis plus O(r^3) work, and ``basis()`` materialises Phi when needed.
    Every update is mathematically tracking.py:141-178; a failed update
    (non-finite snapshot -> ``DenseError``) leaves the stream unchanged.
    """

    def __init__(self, basis: ReducedBasis):
        phi = _dev.dev(basis.phi)
        self.n, self.r = phi.shape
        self._ctx = Context.get()
        h = C.c_void_p()
        self._ctx.call("adrom_isvd_stream_create", C.c_int64(self.n), C.c_int32(self.r), C.byref(h))
        self._h = h
        sig = _dev.dev(basis.sigma)
        self._ctx.scall("adrom_isvd_stream_load", self._h, ptr(phi), ptr(sig))

    def update(self, y_hat, lam: float) -> dict:
        y = _dev.dev(y_hat)
        if y.dim() != 1 or y.shape[0] != self.n:
            raise ValueError(f"snapshot length {tuple(y.shape)} does not match basis rows {self.n}")
        info = IsvdInfo()
        self._ctx.scall("adrom_isvd_stream_update", self._h, ptr(y), C.c_double(lam), C.byref(info))
        return dict(qnorm=info.qnorm, ynorm=info.ynorm, proj_resid=info.proj_resid,
                    degenerate=bool(info.degenerate), sweeps=info.sweeps)

    def basis_sigma(self):
        """The current singular values (device vector, no basis materialisation)."""
        sig = _dev.empty(self.r)
        self._ctx.scall("adrom_isvd_stream_read", self._h, None, ptr(sig))
        return sig

    def basis(self) -> ReducedBasis:
        phi = _dev.empty(self.n, self.r)
        sig = _dev.empty(self.r)
        self._ctx.scall("adrom_isvd_stream_read", self._h, ptr(phi), ptr(sig))
        return ReducedBasis(phi=phi, sigma=sig)

    def close(self):
        if getattr(self, "_h", None):
            self._ctx.lib.adrom_isvd_stream_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
