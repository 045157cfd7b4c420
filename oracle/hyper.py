"""Oracle: hyper-reduction sampling and the sampled-residual gather plan.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Restates ``/root/reference/pkg/src/adrom/sampling.py`` (QDEIM 77-114, FGS
117-159, DEIM pseudo-inverse 162-175, stencil closure 178-189) and
``fom.py:119-158`` (``SamplingPlan``).  QDEIM calls the same LAPACK driver
as the reference (``scipy.linalg.qr(pivoting=True)`` = geqp3); an
exact-greedy restatement is provided next to it because it is the
definition the GPU kernel implements and because geqp3 on a 64 x 2^24
matrix takes minutes.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg

from .physics import Model, OracleDenseError, primitive_fields, rhs_from_stencils
from .subspace import SVD_CUTOFF, thin_svd


def pivot_sequence(mat, count):
    """sampling.py:77-104 — first ``count`` pivots of a restarted
    column-pivoted QR (geqp3) of the r x N matrix ``mat``."""
    n_cols = mat.shape[1]
    if count > n_cols:
        raise OracleDenseError(f"cannot select {count} pivots from {n_cols} columns")
    chosen: list[int] = []
    remaining = np.arange(n_cols)
    while len(chosen) < count:
        _, rr, piv = scipy.linalg.qr(mat[:, remaining], mode="economic", pivoting=True)
        diag = np.abs(np.diag(rr))
        take = min(count - len(chosen), diag.size)
        for j in range(take):
            if diag[j] < 1e-14:
                raise OracleDenseError(
                    f"rank deficiency at pivot step {len(chosen) + j} "
                    f"(residual column norm {diag[j]:.3e})")
            chosen.append(int(remaining[piv[j]]))
        remaining = np.setdiff1d(remaining, np.array(chosen, dtype=int))
    return chosen


def greedy_pivots(phi, count):
    """Exact greedy restatement of the QDEIM pivot rule.

    Rows of ``phi`` (= columns of phi^T) are chosen by largest residual
    norm after projecting out the directions of the rows already chosen
    (modified Gram-Schmidt), ties to the lowest row index (LAPACK
    ``idamax``).  Restarts every ``r`` pivots like ``pivot_sequence``.
    Returns (pivots, residual_norms_at_selection).
    """
    phi = np.asarray(phi, dtype=float)
    n, r = phi.shape
    chosen: list[int] = []
    norms: list[float] = []
    taken = np.zeros(n, dtype=bool)
    while len(chosen) < count:
        work = phi.copy()
        for _ in range(min(r, count - len(chosen))):
            res = np.einsum("ij,ij->i", work, work)
            res[taken] = -1.0
            best = int(np.argmax(res))          # first maximum = lowest index
            nrm = float(np.sqrt(res[best]))
            if nrm < 1e-14:
                raise OracleDenseError(
                    f"rank deficiency at pivot step {len(chosen)} "
                    f"(residual column norm {nrm:.3e})")
            d = work[best] / nrm
            work -= np.outer(work @ d, d)
            chosen.append(best)
            norms.append(nrm)
            taken[best] = True
    return chosen, norms


@dataclass(frozen=True)
class Sampling:
    """sampling.py:30-49 — ordered distinct sampled rows + sorted closure."""

    indices: np.ndarray
    closure: np.ndarray


def qdeim(phi, n_s, exact_greedy=False):
    """sampling.py:107-114."""
    if exact_greedy:
        idx = np.array(greedy_pivots(phi, n_s)[0], dtype=np.int64)
    else:
        idx = np.array(pivot_sequence(np.asarray(phi).T, n_s), dtype=np.int64)
    return Sampling(indices=idx, closure=np.unique(idx))


def feature_field(model: Model, q, kind):
    """sampling.py:64-74 — per-cell feature used by FGS."""
    fields = primitive_fields(model, q)
    names = ("u",) if model.kind == "burgers" else ("rho", "v", "p")
    if kind == "pressure-gradient":
        key = "p" if "p" in fields else names[0]
    elif kind == "velocity-gradient":
        key = "v" if "v" in fields else names[0]
    else:
        raise ValueError(f"unknown feature map {kind!r}")
    return fields[key]


def fgs(phi, y_corr, n_s, n_extra, feature, model: Model, exact_greedy=False):
    """sampling.py:117-159 — QDEIM rows + strongest |grad theta| cells."""
    if n_extra > n_s:
        raise ValueError("n_extra cannot exceed the total number of sampling points")
    n_base = n_s - n_extra
    if n_base > 0:
        base = (greedy_pivots(phi, n_base)[0] if exact_greedy
                else pivot_sequence(np.asarray(phi).T, n_base))
    else:
        base = []
    theta = feature_field(model, y_corr, feature)
    grad = np.empty_like(theta)
    grad[1:-1] = (theta[2:] - theta[:-2]) / (2.0 * model.dx)
    grad[0] = (theta[1] - theta[0]) / model.dx
    grad[-1] = (theta[-1] - theta[-2]) / model.dx
    order = np.lexsort((np.arange(theta.size), -np.abs(grad)))
    picked = list(base)
    seen = set(picked)
    left = n_extra
    for cell in order:
        if left == 0:
            break
        for v in range(model.n_var):
            row = int(cell) * model.n_var + v
            if row in seen:
                continue
            picked.append(row)
            seen.add(row)
            left -= 1
            if left == 0:
                break
    if left > 0:
        raise OracleDenseError("not enough distinct rows to satisfy the sampling budget")
    idx = np.array(picked, dtype=np.int64)
    return Sampling(indices=idx, closure=np.unique(idx))


def closure(sampling: Sampling, model: Model) -> Sampling:
    """sampling.py:178-189 — all variables of sampled cells and neighbours."""
    nv = model.n_var
    cells = np.unique(sampling.indices // nv)
    lft, rgt = model.neighbours(cells)
    every = np.unique(np.concatenate([lft, cells, rgt]))
    rows = (every[:, None] * nv + np.arange(nv)[None, :]).ravel()
    return Sampling(indices=sampling.indices,
                    closure=np.unique(np.concatenate([rows, sampling.indices])))


def deim_pinv(phi, indices):
    """sampling.py:162-175 — (P^T Phi)^+ via thin SVD, shape (r, n_s)."""
    u, s, v = thin_svd(np.asarray(phi)[indices, :])
    if s[-1] <= SVD_CUTOFF * s[0]:
        raise OracleDenseError(
            f"sampled basis is rank deficient (smallest singular value {s[-1]:.3e})")
    return (v / s) @ u.T


@dataclass
class GatherPlan:
    """fom.py:119-158 — closure positions of each sampled cell's stencil."""

    cells: np.ndarray       # (k,) sorted sampled cells
    gather: np.ndarray      # (k, 3, n_var) positions into the closure array
    out_cell: np.ndarray    # (n_s,) sampled row -> cell slot
    out_var: np.ndarray     # (n_s,) sampled row -> variable

    def evaluate(self, model: Model, closure_values):
        """fom.py:154-158."""
        per_cell = rhs_from_stencils(model, np.asarray(closure_values)[self.gather])
        return per_cell[self.out_cell, self.out_var]


def gather_plan(model: Model, sampling: Sampling) -> GatherPlan:
    """fom.py:127-152."""
    nv = model.n_var
    clo = np.asarray(sampling.closure, dtype=np.int64)
    cells = np.unique(sampling.indices // nv)
    lft, rgt = model.neighbours(cells)

    def slots(cs):
        rows = cs[:, None] * nv + np.arange(nv)[None, :]
        at = np.searchsorted(clo, rows)
        at_c = np.minimum(at, clo.size - 1)
        if np.any(clo[at_c] != rows):
            raise ValueError("sampling closure is missing required stencil rows; "
                             "expand it with stencil_closure() first")
        return at_c

    gather = np.stack([slots(lft), slots(cells), slots(rgt)], axis=1)
    out_cell = np.searchsorted(cells, sampling.indices // nv)
    return GatherPlan(cells=cells, gather=gather, out_cell=out_cell,
                      out_var=sampling.indices % nv)
