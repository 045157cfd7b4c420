"""Oracle: reduced operator, encode/decode, LSPG and Galerkin reduced steps.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Restates ``/root/reference/pkg/src/adrom/projection.py`` (``RomOperator``
57-87, ``encode``/``decode`` 96-104, ``galerkin_step`` 111-147,
``lspg_step`` 158-204, ``lspg_objective`` 207-214).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .hyper import GatherPlan, Sampling, deim_pinv, gather_plan
from .physics import FD_EPS, Model


class OracleRomStepError(RuntimeError):
    """projection.py:37-38."""


@dataclass
class Operator:
    """projection.py:57-87 — basis, scaling, sampling and closure caches."""

    phi: np.ndarray
    q_ref: np.ndarray
    row_scale: np.ndarray
    sampling: Sampling
    plan: GatherPlan
    pinv: np.ndarray            # (r, n_s)
    d_sampled: np.ndarray       # (n_s,)
    q_ref_closure: np.ndarray   # (n_c,)
    dinv_phi_closure: np.ndarray  # (n_c, r)
    phi_sampled: np.ndarray     # (n_s, r)
    sample_pos: np.ndarray      # (n_s,)

    @property
    def rank(self):
        return self.phi.shape[1]

    def decode_closure(self, a):
        """projection.py:86-87."""
        return self.q_ref_closure + self.dinv_phi_closure @ a


def build_operator(model: Model, phi, q_ref, row_scale, sampling: Sampling) -> Operator:
    """projection.py:61-80."""
    idx = sampling.indices
    clo = sampling.closure
    return Operator(
        phi=phi, q_ref=q_ref, row_scale=row_scale, sampling=sampling,
        plan=gather_plan(model, sampling), pinv=deim_pinv(phi, idx),
        d_sampled=row_scale[idx], q_ref_closure=q_ref[clo],
        dinv_phi_closure=phi[clo, :] / row_scale[clo][:, None],
        phi_sampled=phi[idx, :], sample_pos=np.searchsorted(clo, idx))


def encode(op: Operator, q):
    """projection.py:96-99 — a = Phi^T D (q - q_ref)."""
    return op.phi.T @ (op.row_scale * (np.asarray(q, dtype=float) - op.q_ref))


def decode(op: Operator, a):
    """projection.py:102-104 with snapshots.py:50-51 — q_ref + (Phi a) / d."""
    return op.q_ref + (op.phi @ a) / op.row_scale


def fd_steps(a):
    """projection.py:107-108."""
    return FD_EPS * np.maximum(1.0, np.abs(a))


@dataclass
class StepOutcome:
    """projection.py:49-54 (``RomStepResult``)."""

    a: np.ndarray
    converged: bool
    iterations: int
    residual_norm: float


def lspg_step(op: Operator, model: Model, a_prev, dt, tol=1e-8, max_iter=10) -> StepOutcome:
    """projection.py:158-204 — Gauss-Newton on the gappy-projected BE
    residual with FD directional derivatives along decoded basis columns."""
    a_prev = np.asarray(a_prev, dtype=float)
    prev_s = op.decode_closure(a_prev)[op.sample_pos]
    r = op.rank
    n_s = op.sampling.indices.size
    a = a_prev.copy()
    it = 0
    gnorm = np.inf
    while it < max_iter:
        qc = op.decode_closure(a)
        fs = op.plan.evaluate(model, qc)
        res_s = op.d_sampled * (qc[op.sample_pos] - prev_s - dt * fs)
        rho = op.pinv @ res_s
        h = fd_steps(a)
        dfs = np.empty((n_s, r))
        for j in range(r):
            dfs[:, j] = (op.plan.evaluate(model, qc + h[j] * op.dinv_phi_closure[:, j]) - fs) / h[j]
        test = op.phi_sampled - dt * (op.d_sampled[:, None] * dfs)
        jac = op.pinv @ test
        grad = jac.T @ rho
        gnorm = float(np.linalg.norm(grad))
        if gnorm <= tol:
            break
        sv = np.linalg.svd(jac, compute_uv=False)
        if sv[-1] <= 1e-14 * sv[0]:
            raise OracleRomStepError(
                f"rank-deficient sampled Jacobian at iteration {it} "
                f"(condition number {sv[0] / max(sv[-1], 1e-300):.3e})")
        delta = np.linalg.lstsq(jac, -rho, rcond=1e-12)[0]
        a = a + delta
        it += 1
    return StepOutcome(a, gnorm <= tol, it, gnorm)


def galerkin_step(op: Operator, model: Model, a_prev, dt, tol=1e-8, max_iter=10) -> StepOutcome:
    """projection.py:111-147 — Newton on a' = a + dt (P^T Phi)^+ P^T D f."""
    a0 = np.asarray(a_prev, dtype=float)

    def reduced_rhs(a):
        return op.pinv @ (op.d_sampled * op.plan.evaluate(model, op.decode_closure(a)))

    r = op.rank
    a = a0.copy()
    g = a - a0 - dt * reduced_rhs(a)
    gn = float(np.linalg.norm(g))
    it = 0
    while gn > tol and it < max_iter:
        h = fd_steps(a)
        jac = np.eye(r)
        fa = reduced_rhs(a)
        for j in range(r):
            ap = a.copy()
            ap[j] += h[j]
            jac[:, j] -= dt * (reduced_rhs(ap) - fa) / h[j]
        try:
            delta = np.linalg.solve(jac, -g)
        except np.linalg.LinAlgError as exc:
            raise OracleRomStepError(f"singular reduced Jacobian at iteration {it}") from exc
        a = a + delta
        g = a - a0 - dt * reduced_rhs(a)
        gn = float(np.linalg.norm(g))
        it += 1
    return StepOutcome(a, gn <= tol, it, gn)


def lspg_objective(op: Operator, model: Model, a_prev, a, dt):
    """projection.py:207-214."""
    prev_s = op.decode_closure(np.asarray(a_prev, dtype=float))[op.sample_pos]
    qc = op.decode_closure(a)
    fs = op.plan.evaluate(model, qc)
    rho = op.pinv @ (op.d_sampled * (qc[op.sample_pos] - prev_s - dt * fs))
    return float(rho @ rho)
