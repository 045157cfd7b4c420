"""Hyper-reduction sampling with the reference signatures (``adrom/sampling.py``).

``qdeim_sample`` / ``fgs_sample`` / ``build_deim_operator`` run on the device
(``adrom_qdeim``, ``adrom_fgs``, ``adrom_deim_operator``).  ``SamplingSet``,
``stencil_closure`` and the host view of ``SamplingPlan`` are index
bookkeeping exactly as in the reference; inside the online loop the same
closure and gather plan are built on the device (``plan_build``).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _dev
from ._lib import Context, ptr

__all__ = ["SamplingSet", "FeatureMap", "SamplingPlan", "qdeim_sample", "fgs_sample",
           "build_deim_operator", "stencil_closure"]

_FEATURES = {"pressure-gradient": 0, "velocity-gradient": 1}


@dataclass(frozen=True)
class SamplingSet:
    """sampling.py:30-49 — ordered distinct sampled rows + closure."""

    indices: np.ndarray
    closure: np.ndarray

    def __post_init__(self):
        idx = np.asarray(_dev.host(self.indices), dtype=int)
        clo = np.asarray(_dev.host(self.closure), dtype=int)
        object.__setattr__(self, "indices", idx)
        object.__setattr__(self, "closure", clo)
        if len(np.unique(idx)) != idx.size:
            raise ValueError("sampling indices must be distinct")
        if not np.all(np.isin(idx, clo)):
            raise ValueError("closure must contain every sampled index")

    @property
    def n_samples(self) -> int:
        return int(self.indices.size)


@dataclass(frozen=True)
class FeatureMap:
    """sampling.py:52-74 (built-in extractors only on the device path)."""

    kind: str | Callable = "pressure-gradient"
    n_extra: int = 0


def qdeim_sample(basis, n_s: int) -> SamplingSet:
    """sampling.py:107-114 — exact-greedy pivoted QR of phi^T on the device."""
    phi = _dev.dev(basis.phi)
    n, r = phi.shape
    idx = _dev.empty(n_s, dtype=_dev.torch().int64)
    Context.get().call("adrom_qdeim", ptr(phi), C.c_int64(n), C.c_int32(r), C.c_int32(n_s), ptr(idx))
    ind = _dev.host(idx)
    return SamplingSet(indices=ind, closure=np.unique(ind))


def fgs_sample(basis, y_corr, n_s: int, feature: FeatureMap, model) -> SamplingSet:
    """sampling.py:117-159 — QDEIM rows + strongest feature-gradient cells."""
    if feature.n_extra > n_s:
        raise ValueError("n_extra cannot exceed the total number of sampling points")
    if callable(feature.kind) or feature.kind not in _FEATURES:
        if callable(feature.kind):
            raise TypeError("callable feature maps have no device implementation")
        raise ValueError(f"unknown feature map {feature.kind!r}")
    phi = _dev.dev(basis.phi)
    r = phi.shape[1]
    y = _dev.dev(y_corr)
    idx = _dev.empty(n_s, dtype=_dev.torch().int64)
    m = model.abi()
    Context.get().call("adrom_fgs", C.byref(m), ptr(phi), C.c_int32(r), ptr(y), C.c_int32(n_s),
                       C.c_int32(feature.n_extra), C.c_int32(_FEATURES[feature.kind]), ptr(idx))
    ind = _dev.host(idx)
    return SamplingSet(indices=ind, closure=np.unique(ind))


def build_deim_operator(basis, sampling: SamplingSet):
    """sampling.py:162-175 — (P^T Phi)^+, shape (r, n_s)."""
    phi = _dev.dev(basis.phi)
    n, r = phi.shape
    idx = _dev.dev_i64(sampling.indices)
    n_s = int(idx.numel())
    out = _dev.empty(r, n_s)
    Context.get().call("adrom_deim_operator", ptr(phi), C.c_int64(n), C.c_int32(r), ptr(idx),
                       C.c_int32(n_s), ptr(out))
    return _dev.like(out, basis.phi)


def stencil_closure(sampling: SamplingSet, model) -> SamplingSet:
    """sampling.py:178-189 (index bookkeeping, as in the reference)."""
    nv = model.n_var
    cells = np.unique(sampling.indices // nv)
    left, right = model.neighbor_cells(cells)
    every = np.unique(np.concatenate([left, cells, right]))
    rows = (every[:, None] * nv + np.arange(nv)[None, :]).ravel()
    closure = np.unique(np.concatenate([rows, sampling.indices]))
    return SamplingSet(indices=sampling.indices, closure=closure)


class SamplingPlan:
    """fom.py:119-158 — gather map; ``evaluate`` runs ``adrom_plan_evaluate``."""

    def __init__(self, model, sampling: SamplingSet):
        self.model = model
        self.closure = np.asarray(sampling.closure, dtype=int)
        nv = model.n_var
        cells = np.unique(np.asarray(sampling.indices, dtype=int) // nv)
        left, right = model.neighbor_cells(cells)
        pos = {int(row): i for i, row in enumerate(self.closure)}

        def rows_of(cs):
            try:
                return np.array([[pos[int(c) * nv + v] for v in range(nv)] for c in cs], dtype=int)
            except KeyError as exc:
                raise ValueError("sampling closure is missing required stencil rows; "
                                 "expand it with stencil_closure() first") from exc

        self._cells = cells
        self._gather = np.stack([rows_of(left), rows_of(cells), rows_of(right)], axis=1)
        cell_pos = {int(c): i for i, c in enumerate(cells)}
        idx = np.asarray(sampling.indices, dtype=int)
        self._out_cell = np.array([cell_pos[int(i) // nv] for i in idx], dtype=int)
        self._out_var = idx % nv
        self._dev = None

    def _device(self):
        if self._dev is None:
            self._dev = (_dev.dev_i64(self._gather), _dev.dev_i64(self._out_cell),
                         _dev.dev_i64(self._out_var))
        return self._dev

    def evaluate(self, closure_values, h=None, dirs=None):
        """Rhs at the sampled rows (fom.py:154-158).  With ``h`` (n_dir,) and
        ``dirs`` (n_closure, ld) returns (n_dir, n_s) for values
        ``closure_values + h[d] * dirs[:, d]`` (projection.py:185)."""
        g, oc, ov = self._device()
        cv = _dev.dev(closure_values)
        n_s = int(oc.numel())
        m = self.model.abi()
        if h is None:
            out = _dev.empty(n_s)
            Context.get().call("adrom_plan_evaluate", C.byref(m), ptr(g), C.c_int64(g.shape[0]),
                               ptr(oc), ptr(ov), C.c_int64(n_s), ptr(cv), None, None,
                               C.c_int64(0), C.c_int32(0), ptr(out))
            return _dev.like(out, closure_values)
        hd, dd = _dev.dev(h), _dev.dev(dirs)
        nd = int(hd.numel())
        out = _dev.empty(nd, n_s)
        Context.get().call("adrom_plan_evaluate", C.byref(m), ptr(g), C.c_int64(g.shape[0]),
                           ptr(oc), ptr(ov), C.c_int64(n_s), ptr(cv), ptr(hd), ptr(dd),
                           C.c_int64(dd.shape[1]), C.c_int32(nd), ptr(out))
        return _dev.like(out, closure_values)
