"""Oracle: full-order residuals, banded FD Jacobian and backward-Euler Newton.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Restates ``/root/reference/pkg/src/adrom/fom.py`` and ``dense.py:newton_solve``
with the Jacobian stored as 3 blocks per cell row instead of a dense N x N
matrix (the reference's dense matrix is O(N^2): 2.25 PB at N = 2^24).  The
block entries are the reference's entries bit for bit: row i of ``rhs``
depends only on cells i-1, i, i+1 (``fom.py:305-309``) and the reference
perturbs cells of one stencil colour together (``fom.py:318-327``), so each
entry is ``(rhs_i(q + eps_j e_j) - rhs_i(q)) / eps_j`` evaluated with the
very same floating-point operations.

Floating-point order is mirrored operation by operation (numpy never
contracts to FMA), e.g. ``(um - 2.0*u) + up`` then ``nu*(...)/dx**2``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg
import scipy.sparse
import scipy.sparse.linalg

#: density / pressure floor of the primitive recovery (fom.py:36)
PRIM_FLOOR = 1e-10
#: finite-difference perturbation scale (fom.py:39)
FD_EPS = 1e-7


@dataclass(frozen=True)
class Model:
    """Minimal model descriptor (kind + grid + physics constants).

    Mirrors the fields of ``BurgersProblem`` (fom.py:161-174) and
    ``SodProblem`` (fom.py:249-260) that the residual needs.
    """

    kind: str           # "burgers" | "sod" | "reacting" (configuration 4, oracle/reacting.py)
    n_elem: int
    nu: float = 0.01
    gamma: float = 1.4
    length: float = 1.0
    mech: tuple | None = None  # reacting: the (5, 12) mechanism, flattened

    @property
    def n_var(self) -> int:
        return {"burgers": 1, "sod": 3, "reacting": 13}[self.kind]

    @property
    def periodic(self) -> bool:
        return self.kind in ("burgers", "reacting")

    @property
    def dx(self) -> float:
        # fom.py:74  dx = length / n_elem
        return self.length / self.n_elem

    @property
    def n_dof(self) -> int:
        return self.n_var * self.n_elem

    def neighbours(self, cells):
        """fom.py:92-97 — wrap for periodic, clamp otherwise."""
        cells = np.asarray(cells, dtype=np.int64)
        if self.periodic:
            return (cells - 1) % self.n_elem, (cells + 1) % self.n_elem
        return np.maximum(cells - 1, 0), np.minimum(cells + 1, self.n_elem - 1)


# --------------------------------------------------------------------------
# pointwise physics
# --------------------------------------------------------------------------

def burgers_point(um, u, up, dx, nu):
    """Burgers cell residual from (left, centre, right) values.

    fom.py:184-188 (and the identical gather form fom.py:194-198):
    sign-dependent first-order upwind convection in non-conservative form
    plus centred diffusion.
    """
    back = (u - um) / dx
    fwd = (up - u) / dx
    conv = -u * np.where(u > 0.0, back, fwd)
    lap = (um - 2.0 * u) + up
    diff = nu * lap / dx ** 2
    return conv + diff


def euler_primitives(cons, gamma):
    """fom.py:204-210 — floored density / pressure recovery."""
    rho = np.maximum(cons[..., 0], PRIM_FLOOR)
    vel = cons[..., 1] / rho
    kinetic = 0.5 * rho * vel ** 2
    p = np.maximum((gamma - 1.0) * (cons[..., 2] - kinetic), PRIM_FLOOR)
    return rho, vel, p


def euler_flux(cons, gamma):
    """fom.py:213-219 — physical Euler flux of conserved triplets."""
    rho, vel, p = euler_primitives(cons, gamma)
    out = np.empty_like(cons)
    out[..., 0] = cons[..., 1]
    out[..., 1] = cons[..., 1] * vel + p
    out[..., 2] = vel * (cons[..., 2] + p)
    return out


def rusanov(left, right, gamma):
    """fom.py:222-236 — local Lax-Friedrichs interface flux."""
    left = np.asarray(left, dtype=float)
    right = np.asarray(right, dtype=float)
    rl, vl, pl = euler_primitives(left, gamma)
    rr, vr, pr = euler_primitives(right, gamma)
    speed = np.maximum(np.abs(vl) + np.sqrt(gamma * pl / rl),
                       np.abs(vr) + np.sqrt(gamma * pr / rr))
    avg = 0.5 * (euler_flux(left, gamma) + euler_flux(right, gamma))
    return avg - 0.5 * speed[..., None] * (right - left)


# --------------------------------------------------------------------------
# full residuals
# --------------------------------------------------------------------------

def rhs(model: Model, q: np.ndarray) -> np.ndarray:
    """Semi-discrete right-hand side f(q) on the interleaved layout.

    Burgers: fom.py:180-188 (periodic via roll).
    Sod:     fom.py:265-269 (ghost copies at both ends, Rusanov fluxes at
             the n+1 interfaces, flux difference over dx).
    """
    q = np.asarray(q, dtype=float)
    if model.kind == "burgers":
        return burgers_point(np.roll(q, 1), q, np.roll(q, -1), model.dx, model.nu)
    if model.kind == "sod":
        cells = q.reshape(model.n_elem, 3)
        ext = np.concatenate([cells[:1], cells, cells[-1:]], axis=0)
        face = rusanov(ext[:-1], ext[1:], model.gamma)
        return (-(face[1:] - face[:-1]) / model.dx).ravel()
    if model.kind == "reacting":
        from . import reacting
        mech = np.asarray(model.mech, dtype=float).reshape(5, reacting.N_REACT)
        return reacting.rhs(q, model.n_elem, model.dx, model.gamma, mech)
    raise ValueError(f"unknown model kind {model.kind!r}")


def rhs_from_stencils(model: Model, stencil: np.ndarray) -> np.ndarray:
    """Residual at k cells from gathered (left, centre, right) states.

    ``stencil`` has shape (k, 3, n_var); returns (k, n_var).
    Burgers: fom.py:190-198.  Sod: fom.py:271-277.  Reacting (configuration
    4, oracle/reacting.py): Rusanov faces of the 13-variable state plus the
    centre cell's sources.
    """
    if model.kind == "burgers":
        val = burgers_point(stencil[:, 0, 0], stencil[:, 1, 0], stencil[:, 2, 0],
                            model.dx, model.nu)
        return val[:, None]
    if model.kind == "sod":
        lo = rusanov(stencil[:, 0, :], stencil[:, 1, :], model.gamma)
        hi = rusanov(stencil[:, 1, :], stencil[:, 2, :], model.gamma)
        return -(hi - lo) / model.dx
    if model.kind == "reacting":  # oracle/reacting.py: the same faces and sources as rhs()
        from . import reacting
        mech = np.asarray(model.mech, dtype=float).reshape(5, reacting.N_REACT)
        lo = reacting.rusanov(stencil[:, 0, :], stencil[:, 1, :], model.gamma)
        hi = reacting.rusanov(stencil[:, 1, :], stencil[:, 2, :], model.gamma)
        return -(hi - lo) / model.dx + reacting.sources(stencil[:, 1, :], model.gamma, mech)
    raise ValueError(f"unknown model kind {model.kind!r}")


# --------------------------------------------------------------------------
# banded finite-difference Jacobian
# --------------------------------------------------------------------------

def colour_classes(model: Model) -> list[np.ndarray]:
    """fom.py:285-298 — cells that may be perturbed together (mod-3
    striping, tail fix for periodic grids whose size is not a multiple of 3)."""
    n = model.n_elem
    tag = np.arange(n) % 3
    if model.periodic and n % 3 == 1:
        tag[n - 1] = 3
    elif model.periodic and n % 3 == 2:
        tag[n - 2] = 3
        tag[n - 1] = 4
    return [np.flatnonzero(tag == t) for t in range(int(tag.max()) + 1)]


def fd_eps(q: np.ndarray) -> np.ndarray:
    """fom.py:317 — eps_j = 1e-7 * max(1, |q_j|)."""
    return FD_EPS * np.maximum(1.0, np.abs(q))


def fd_jacobian_blocks(model: Model, q: np.ndarray, f0: np.ndarray | None = None) -> np.ndarray:
    """Block-tridiagonal FD Jacobian, shape (n_elem, 3, n_var, n_var).

    ``B[i, 0]`` = d rhs_i / d q_{left(i)}, ``B[i, 1]`` = d rhs_i / d q_i,
    ``B[i, 2]`` = d rhs_i / d q_{right(i)}; for clamped boundaries the
    missing neighbour block of the end cells is zero (its derivative is in
    the centre block, exactly as ``np.unique`` collapses rows in
    fom.py:325).  Entries are those of ``fd_jacobian`` (fom.py:301-328).
    """
    q = np.asarray(q, dtype=float)
    nv, n = model.n_var, model.n_elem
    base = rhs(model, q) if f0 is None else f0
    eps = fd_eps(q)
    blocks = np.zeros((n, 3, nv, nv))
    for cells in colour_classes(model):
        lft, rgt = model.neighbours(cells)
        for v in range(nv):
            cols = cells * nv + v
            pert = q.copy()
            pert[cols] += eps[cols]
            delta = (rhs(model, pert) - base).reshape(n, nv)
            e = eps[cols][:, None]
            # column (cell c, var v) touches rows of cells left(c), c, right(c)
            blocks[cells, 1, :, v] = delta[cells] / e
            if model.periodic:
                blocks[rgt, 0, :, v] = delta[rgt] / e      # row right(c), left block
                blocks[lft, 2, :, v] = delta[lft] / e      # row left(c), right block
            else:
                inner_r = rgt != cells
                inner_l = lft != cells
                blocks[rgt[inner_r], 0, :, v] = delta[rgt[inner_r]] / e[inner_r]
                blocks[lft[inner_l], 2, :, v] = delta[lft[inner_l]] / e[inner_l]
    return blocks


def blocks_to_dense(model: Model, blocks: np.ndarray) -> np.ndarray:
    """Expand block-tridiagonal storage to the reference's dense layout."""
    nv, n = model.n_var, model.n_elem
    dense = np.zeros((n * nv, n * nv))
    cells = np.arange(n)
    lft, rgt = model.neighbours(cells)
    for i in range(n):
        rows = slice(i * nv, (i + 1) * nv)
        if lft[i] != i:
            dense[rows, lft[i] * nv:(lft[i] + 1) * nv] = blocks[i, 0]
        dense[rows, i * nv:(i + 1) * nv] = blocks[i, 1]
        if rgt[i] != i:
            dense[rows, rgt[i] * nv:(rgt[i] + 1) * nv] = blocks[i, 2]
    return dense


def newton_matrix(model: Model, blocks: np.ndarray, dt: float) -> scipy.sparse.csc_matrix:
    """Sparse ``I - dt * J`` (fom.py:343-344) from block storage."""
    nv, n = model.n_var, model.n_elem
    cells = np.arange(n)
    lft, rgt = model.neighbours(cells)
    rows, cols, vals = [], [], []
    ii, jj = np.meshgrid(np.arange(nv), np.arange(nv), indexing="ij")
    for slot, nb in ((0, lft), (1, cells), (2, rgt)):
        keep = np.ones(n, dtype=bool) if slot == 1 else (nb != cells)
        c = cells[keep]
        r_idx = (c[:, None, None] * nv + ii[None]).ravel()
        c_idx = (nb[keep][:, None, None] * nv + jj[None]).ravel()
        vals.append((-dt * blocks[keep, slot]).ravel())
        rows.append(r_idx)
        cols.append(c_idx)
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    vals = np.concatenate(vals)
    diag = rows == cols
    vals = vals.copy()
    # eye - dt*J: diagonal entries are 1.0 - dt*J_ii, off-diagonals 0.0 - dt*J_ij
    vals[diag] = 1.0 - (-vals[diag])
    return scipy.sparse.csc_matrix((vals, (rows, cols)), shape=(n * nv, n * nv))


def _cyclic_tridiag_solve(model: Model, blocks: np.ndarray, dt: float, rhs_vec: np.ndarray):
    """Solve ``(I - dt J) x = rhs`` for a scalar periodic model (cyclic
    tridiagonal) by Sherman-Morrison around LAPACK's banded solver (gbsv).

    Used beyond 2^20 cells, where SuperLU's workspace overflows (it fails at
    2^24, configuration 3).  Same matrix entries as ``newton_matrix``; the
    solve rounds differently at the 1e-16 level, like the sparse LU does
    against the reference's dense LU."""
    n = model.n_elem
    sub = -dt * blocks[:, 0, 0, 0]       # A[i, i-1] (row i)
    diag = 1.0 - dt * blocks[:, 1, 0, 0]
    sup = -dt * blocks[:, 2, 0, 0]       # A[i, i+1]
    alpha = sup[n - 1]                   # A[n-1, 0]
    beta = sub[0]                        # A[0, n-1]
    gamma = -diag[0]
    ab = np.zeros((3, n))
    ab[0, 1:] = sup[:-1]
    ab[1] = diag
    ab[1, 0] = diag[0] - gamma
    ab[1, n - 1] = diag[n - 1] - alpha * beta / gamma
    ab[2, :-1] = sub[1:]
    u = np.zeros(n)
    u[0], u[n - 1] = gamma, alpha
    ys = scipy.linalg.solve_banded((1, 1), ab, np.column_stack([rhs_vec, u]),
                                   overwrite_ab=True, check_finite=False)
    y, zz = ys[:, 0], ys[:, 1]
    fac = (y[0] + beta / gamma * y[n - 1]) / (1.0 + zz[0] + beta / gamma * zz[n - 1])
    return y - fac * zz


@dataclass
class NewtonOutcome:
    """Mirror of ``dense.NewtonResult`` (dense.py:129-137)."""

    x: np.ndarray
    converged: bool
    iterations: int
    residual_norm: float


class OracleDenseError(RuntimeError):
    """Mirror of ``dense.DenseError`` (dense.py:35-36)."""


def implicit_step(model: Model, q: np.ndarray, dt: float, tol: float = 1e-8,
                  max_iter: int = 10) -> NewtonOutcome:
    """Backward Euler ``x - q - dt f(x) = 0`` by Newton.

    fom.py:331-347 + dense.py:140-171: absolute stop ``||r||_2 <= tol``
    checked before each Jacobian, at most ``max_iter`` updates,
    non-convergence flagged, non-finite residual raises.  The linear solve
    is a sparse LU of the block-tridiagonal ``I - dt J`` instead of the
    reference's dense LU (same matrix entries; rounding of the solve
    differs at the 1e-16 level).
    """
    if tol <= 0:
        raise OracleDenseError("newton_solve requires tol > 0")
    q = np.asarray(q, dtype=float)
    x = q.copy()

    def residual(xx):
        val = xx - q - dt * rhs(model, xx)
        if not np.all(np.isfinite(val)):
            raise OracleDenseError("newton residual contains non-finite entries")
        return val

    r = residual(x)
    rn = float(np.linalg.norm(r))
    for it in range(max_iter):
        if rn <= tol:
            return NewtonOutcome(x, True, it, rn)
        blocks = fd_jacobian_blocks(model, x)
        if not np.all(np.isfinite(blocks)):
            raise OracleDenseError("newton jacobian contains non-finite entries")
        if model.n_var == 1 and model.periodic and model.n_elem > (1 << 20):
            x = x + _cyclic_tridiag_solve(model, blocks, dt, -r)
            r = residual(x)
            rn = float(np.linalg.norm(r))
            continue
        mat = newton_matrix(model, blocks, dt)
        try:
            lu = scipy.sparse.linalg.splu(mat, permc_spec="NATURAL",
                                          diag_pivot_thresh=1.0)
        except RuntimeError as exc:  # dense.py:163-166
            raise OracleDenseError(f"singular Jacobian at Newton iteration {it}") from exc
        x = x + lu.solve(-r)
        r = residual(x)
        rn = float(np.linalg.norm(r))
    return NewtonOutcome(x, rn <= tol, max_iter, rn)


def coarse_step(model: Model, y: np.ndarray, z: int, dt: float, tol: float = 1e-8,
                max_iter: int = 10) -> NewtonOutcome:
    """fom.py:350-356 — implicit step of size z*dt."""
    if z < 1:
        raise ValueError("z must be at least 1")
    return implicit_step(model, y, z * dt, tol, max_iter)


def sod_state(n_elem: int, gamma: float = 1.4) -> np.ndarray:
    """fom.py:239-246 — Sod Riemann data, interleaved conserved state."""
    x = (np.arange(n_elem) + 0.5) / n_elem
    rho = np.where(x < 0.5, 1.0, 0.125)
    p = np.where(x < 0.5, 1.0, 0.1)
    vel = np.zeros(n_elem)
    energy = p / (gamma - 1.0) + 0.5 * rho * vel ** 2
    return np.stack([rho, rho * vel, energy], axis=1).ravel()


def primitive_fields(model: Model, q: np.ndarray) -> dict:
    """fom.py:200-201 / 279-282."""
    if model.kind == "burgers":
        return {"u": np.asarray(q, dtype=float)}
    cells = np.asarray(q, dtype=float).reshape(model.n_elem, model.n_var)[:, :3]
    rho, vel, p = euler_primitives(cells, model.gamma)
    return {"rho": rho, "v": vel, "p": p}
