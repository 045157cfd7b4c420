"""Scaling and offline POD with the reference signatures (``adrom/snapshots.py``).

Preprocess/lift are elementwise and run where the data lives; ``fit_scaling``
and ``pod`` are the OFFLINE stage (outside the timed region, SURVEY §8f item
2) and run on the library's own kernels: a fixed-order reduction for the
scales, Householder QR of the snapshot matrix (or of its transpose when the
window is wider than the grid) + one-sided Jacobi SVD of the triangular
factor + Q application + fix_column_signs (csrc/hhqr.cu, csrc/offline.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

import ctypes as C

from . import _dev
from ._lib import Context, ptr
from .errors import DenseError
from .tracking import ReducedBasis

__all__ = ["ScalingTransform", "fit_scaling", "pod", "pod_window", "VAR_FLOOR"]

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
    """snapshots.py:54-69 (adrom_fit_scaling)."""
    if len(training) < 1:
        raise ValueError("need at least one training snapshot")
    t = _dev.torch()
    first = training[0]
    dev = _dev.is_device(first)
    tr = training if (_dev.is_device(training) and training.dim() == 2) else \
        t.stack([_dev.dev(q) for q in training])
    tr = tr.contiguous()
    m, n = tr.shape
    q_ref = _dev.empty(n)
    phi_norm = _dev.empty(n_var)
    Context.get().call("adrom_fit_scaling", ptr(tr), C.c_int32(m), C.c_int64(n), C.c_int32(n_var),
                       ptr(q_ref), ptr(phi_norm))
    if dev:
        return ScalingTransform(q_ref=q_ref, phi_norm=phi_norm)
    return ScalingTransform(q_ref=_dev.host(q_ref), phi_norm=_dev.host(phi_norm))


def pod(snapshots, r: int) -> ReducedBasis:
    """snapshots.py:72-89 — leading r left singular vectors, sign-fixed, with
    the numerical-rank check (adrom_pod)."""
    y = _dev.dev(snapshots)
    if y.dim() != 2:
        raise ValueError("snapshot matrix must be 2-d (one column per snapshot)")
    n, m = y.shape
    if r > min(n, m):
        raise DenseError(f"cannot extract {r} modes from a {n}x{m} matrix")
    phi = _dev.empty(n, r)
    sigma = _dev.empty(r)
    rank = C.c_int32(0)
    Context.get().call("adrom_pod", ptr(y), C.c_int64(n), C.c_int32(m), C.c_int32(r), ptr(phi),
                       ptr(sigma), None, C.byref(rank))
    return ReducedBasis(phi=_dev.like(phi, snapshots), sigma=_dev.like(sigma, snapshots))


def pod_window(training, scaling: ScalingTransform, r: int) -> ReducedBasis:
    """pod(column_stack(preprocess(q) for q in training), r) without forming
    the N x m snapshot matrix twice (driver.py:298-299; adrom_pod_window)."""
    tr = _dev.dev(training).contiguous()
    m, n = tr.shape
    nv = scaling.n_var
    phi = _dev.empty(n, r)
    sigma = _dev.empty(r)
    rank = C.c_int32(0)
    if r > min(n, m):
        raise DenseError(f"cannot extract {r} modes from a {n}x{m} matrix")
    q_ref, phi_norm = _dev.dev(scaling.q_ref), _dev.dev(scaling.phi_norm)  # alive across the call
    Context.get().call("adrom_pod_window", ptr(tr), C.c_int32(m), C.c_int64(n), C.c_int32(nv),
                       ptr(q_ref), ptr(phi_norm), C.c_int32(r),
                       ptr(phi), ptr(sigma), None, C.byref(rank))
    return ReducedBasis(phi=phi, sigma=sigma)
