"""Scaling and offline POD with the reference signatures (``adrom/snapshots.py``).

Preprocess/lift are elementwise and run where the data lives; ``pod`` is the
OFFLINE stage (outside the timed region) and uses a
QR + small SVD (torch/cuSOLVER for the QR; the one-block Jacobi SVD of the
CUDA library for the small triangular factor when it fits, cuSOLVER
otherwise).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev
from .errors import DenseError
from .tracking import ReducedBasis

__all__ = ["ScalingTransform", "fit_scaling", "pod", "VAR_FLOOR"]

VAR_FLOOR = 1e-30  # snapshots.py:23


@dataclass(frozen=True)
class ScalingTransform:
    """snapshots.py:26-51."""

    q_ref: object
    phi_norm: object

    @property
    def n_var(self) -> int:
        return int(np.asarray(_dev.host(self.phi_norm)).size)

    @property
    def row_scale(self):
        n_elem = int(self.q_ref.shape[0]) // self.n_var
        if _dev.is_device(self.q_ref):
            pn = _dev.dev(self.phi_norm)
            return (1.0 / pn).repeat(n_elem)
        return np.tile(1.0 / np.asarray(self.phi_norm, dtype=float), n_elem)

    def preprocess(self, q):
        return self.row_scale * (q - self.q_ref)

    def lift(self, y_hat):
        return self.q_ref + y_hat / self.row_scale


def fit_scaling(training, n_var: int) -> ScalingTransform:
    """snapshots.py:54-69."""
    if len(training) < 1:
        raise ValueError("need at least one training snapshot")
    t = _dev.torch()
    first = training[0]
    dev = _dev.is_device(first)
    tr = t.stack([_dev.dev(q) for q in training])
    q_ref = tr[0].clone()
    fluct = tr - q_ref
    per_var = fluct.reshape(len(training), -1, n_var) ** 2
    phi_norm = t.clamp_min(per_var.mean(dim=(0, 1)), VAR_FLOOR)
    phi_norm = t.where(phi_norm <= VAR_FLOOR, t.ones_like(phi_norm), phi_norm)
    if dev:
        return ScalingTransform(q_ref=q_ref, phi_norm=phi_norm)
    return ScalingTransform(q_ref=_dev.host(q_ref), phi_norm=_dev.host(phi_norm))


def _fix_column_signs(q):
    """dense.py:182-189."""
    t = _dev.torch()
    lead = q.abs().argmax(dim=0)
    signs = t.sign(q[lead, t.arange(q.shape[1], device=q.device)])
    signs = t.where(signs == 0, t.ones_like(signs), signs)
    return q * signs


def pod(snapshots, r: int) -> ReducedBasis:
    """snapshots.py:72-89 — leading r left singular vectors, sign-fixed, with
    the numerical-rank check (offline stage)."""
    t = _dev.torch()
    y = _dev.dev(snapshots)
    if y.dim() != 2:
        raise ValueError("snapshot matrix must be 2-d (one column per snapshot)")
    n, m = y.shape
    if r > min(n, m):
        raise DenseError(f"cannot extract {r} modes from a {n}x{m} matrix")
    if not bool(t.isfinite(y).all()):
        raise DenseError("thin_svd input contains non-finite entries")
    if n >= m:
        q, rr = t.linalg.qr(y)
        if m <= 120:
            from .dense import thin_svd
            res = thin_svd(rr)
            ur, s = res.u, res.s
        else:
            ur, s, _ = t.linalg.svd(rr)
        u = q @ ur
    else:
        u, s, _ = t.linalg.svd(y, full_matrices=False)
    rank = int((s > 1e-12 * s[0]).sum()) if float(s[0]) > 0 else 0
    if r > rank:
        raise DenseError(f"requested {r} modes but snapshot matrix has numerical rank {rank}")
    phi = _fix_column_signs(u[:, :r]).contiguous()
    sigma = s[:r].clone().contiguous()
    return ReducedBasis(phi=_dev.like(phi, snapshots), sigma=_dev.like(sigma, snapshots))
