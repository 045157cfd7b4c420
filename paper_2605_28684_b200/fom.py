"""GPU-backed full-order models with the reference ``FomProblem`` surface.

Mirrors ``/root/reference/pkg/src/adrom/fom.py``: ``BurgersProblem``
(fom.py:161-201), ``SodProblem`` (fom.py:249-282), ``TimeStepper``
(fom.py:42-53), ``implicit_step`` / ``coarse_step`` (fom.py:331-356),
``fd_jacobian`` (fom.py:301-328).  Every residual, Jacobian and Newton
solve runs in the CUDA library (``adrom_rhs``, ``adrom_fd_jacobian_blocks``,
``adrom_implicit_step``); topology helpers (neighbour indices, cell
centres) stay on the host like the reference's.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _dev
from ._lib import BURGERS, REACTING, SOD, Context, Model, NewtonInfo, ptr
from .errors import DenseError

__all__ = ["TimeStepper", "FomProblem", "BurgersProblem", "SodProblem", "ReactingEulerProblem",
           "rusanov_flux",
           "reacting_mechanism", "NewtonResult",
           "fd_jacobian", "fd_jacobian_blocks", "implicit_step", "coarse_step",
           "sod_initial_state", "PRIM_FLOOR", "FD_EPS"]

PRIM_FLOOR = 1e-10   # fom.py:36
FD_EPS = 1e-7        # fom.py:39


@dataclass(frozen=True)
class TimeStepper:
    """fom.py:42-53 — backward-Euler settings."""

    dt: float
    newton_tol: float = 1e-8
    newton_max_iter: int = 10

    def __post_init__(self):
        if self.dt <= 0:
            raise ValueError("dt must be positive")


@dataclass
class NewtonResult:
    """dense.py:129-137."""

    x: object
    converged: bool
    iterations: int
    residual_norm: float


class FomProblem:
    """fom.py:56-116 — common surface of the device-backed models."""

    n_var: int = 1
    boundary: str = "periodic"
    stencil_radius: int = 1
    var_names: tuple[str, ...] = ()
    kind: int = 0

    def __init__(self, n_elem: int, length: float = 1.0):
        if n_elem < 4:
            raise ValueError("n_elem must be at least 4")
        self.n_elem = int(n_elem)
        self.length = float(length)
        self.dx = self.length / self.n_elem

    @property
    def n_dof(self) -> int:
        return self.n_var * self.n_elem

    @property
    def cell_centers(self) -> np.ndarray:
        return (np.arange(self.n_elem) + 0.5) * self.dx

    def abi(self) -> Model:
        mech = getattr(self, "_mech_dev", None)
        return Model(self.kind, self.n_var, self.n_elem, self.dx,
                     getattr(self, "nu", 0.0), getattr(self, "gamma", 1.4), ptr(mech))

    def neighbor_cells(self, cells):
        """fom.py:92-97."""
        cells = np.asarray(cells, dtype=int)
        if self.boundary == "periodic":
            return (cells - 1) % self.n_elem, (cells + 1) % self.n_elem
        return np.maximum(cells - 1, 0), np.minimum(cells + 1, self.n_elem - 1)

    # -- residual (kernel 1) ------------------------------------------------
    def rhs(self, q):
        """f(q) on the device (bitwise equal to the reference's numpy)."""
        qd = _dev.dev(q)
        if qd.numel() != self.n_dof:
            raise ValueError(f"state length {qd.numel()} != n_dof {self.n_dof}")
        out = _dev.empty(self.n_dof)
        m = self.abi()
        Context.get().call("adrom_rhs", C.byref(m), ptr(qd), ptr(out))
        return _dev.like(out, q)

    def rhs_at_cells(self, gathered):
        """fom.py:104-110 — (k, 3, n_var) stencils -> (k, n_var)."""
        g = _dev.dev(gathered)
        if g.dim() != 3 or g.shape[1] != 3 or g.shape[2] != self.n_var:
            raise ValueError(f"gathered must have shape (k, 3, {self.n_var})")
        k = g.shape[0]
        out = _dev.empty(k, self.n_var)
        m = self.abi()
        Context.get().call("adrom_rhs_at_cells", C.byref(m), ptr(g), C.c_int64(k), ptr(out))
        return _dev.like(out, gathered)

    def sampling_plan(self, sampling):
        from .sampling import SamplingPlan
        return SamplingPlan(self, sampling)

    def primitive_fields(self, q):
        raise NotImplementedError

    def initial_state(self):
        raise NotImplementedError


class BurgersProblem(FomProblem):
    """fom.py:161-201 — viscous Burgers, periodic, upwind convection."""

    n_var = 1
    boundary = "periodic"
    var_names = ("u",)
    kind = BURGERS

    def __init__(self, n_elem: int, nu: float = 0.01, length: float = 1.0, ic_width: float = 0.1):
        super().__init__(n_elem, length)
        if nu <= 0:
            raise ValueError("viscosity must be positive")
        self.nu = float(nu)
        self.ic_width = float(ic_width)

    def initial_state(self) -> np.ndarray:
        """fom.py:176-178 (host-generated input data)."""
        x = self.cell_centers
        return np.exp(-0.5 * ((x - 0.5 * self.length) / self.ic_width) ** 2)

    def primitive_fields(self, q):
        return {"u": q}


def rusanov_flux(ul, ur, gamma: float):
    """fom.py:222-236 — local Lax-Friedrichs interface flux of single
    conserved triplets or batches (..., 3), bitwise the reference's
    (adrom_rusanov_flux)."""
    uld, urd = _dev.dev(ul), _dev.dev(ur)
    if uld.shape != urd.shape or uld.shape[-1] != 3:
        raise ValueError(f"interface states must have shape (..., 3), got {tuple(uld.shape)}")
    shape = uld.shape
    flat_l, flat_r = uld.reshape(-1, 3).contiguous(), urd.reshape(-1, 3).contiguous()
    out = _dev.empty(flat_l.shape[0], 3)
    Context.get().call("adrom_rusanov_flux", ptr(flat_l), ptr(flat_r), C.c_int64(flat_l.shape[0]),
                       C.c_double(gamma), ptr(out))
    return _dev.like(out.reshape(shape), ul)


def sod_initial_state(n_elem: int, gamma: float = 1.4) -> np.ndarray:
    """fom.py:239-246 (host-generated input data)."""
    x = (np.arange(n_elem) + 0.5) / n_elem
    rho = np.where(x < 0.5, 1.0, 0.125)
    p = np.where(x < 0.5, 1.0, 0.1)
    u = np.zeros(n_elem)
    return np.stack([rho, rho * u, p / (gamma - 1.0) + 0.5 * rho * u ** 2], axis=1).ravel()


class SodProblem(FomProblem):
    """fom.py:249-282 — 1D Euler, Rusanov flux, zero-gradient ghosts."""

    n_var = 3
    boundary = "zero-gradient"
    var_names = ("rho", "v", "p")
    kind = SOD

    def __init__(self, n_elem: int, gamma: float = 1.4, length: float = 1.0):
        super().__init__(n_elem, length)
        if gamma <= 1.0:
            raise ValueError("gamma must exceed 1")
        self.gamma = float(gamma)

    def initial_state(self) -> np.ndarray:
        return sod_initial_state(self.n_elem, self.gamma)

    def primitive_fields(self, q):
        """fom.py:279-282 (diagnostics; evaluated where q lives)."""
        if _dev.is_device(q):
            t = _dev.torch()
            u = q.reshape(self.n_elem, 3)
            rho = t.clamp_min(u[:, 0], PRIM_FLOOR)
            vel = u[:, 1] / rho
            p = t.clamp_min((self.gamma - 1.0) * (u[:, 2] - 0.5 * rho * vel ** 2), PRIM_FLOOR)
            return {"rho": rho, "v": vel, "p": p}
        u = np.asarray(q, dtype=float).reshape(self.n_elem, 3)
        rho = np.maximum(u[:, 0], PRIM_FLOOR)
        vel = u[:, 1] / rho
        p = np.maximum((self.gamma - 1.0) * (u[:, 2] - 0.5 * rho * vel ** 2), PRIM_FLOOR)
        return {"rho": rho, "v": vel, "p": p}


N_SPECIES, N_REACT = 10, 12


def reacting_mechanism(seed: int = 4) -> np.ndarray:
    """Seeded configuration-4 mechanism (SURVEY §8d cfg 4), shape (5, 12):
    reactant a_j, product b_j, A_j = 10**U[8,12] * 1e-10, Ta_j = U[5e3,2e4]/1e3,
    q_j = U[1e5,1e6]/1e6 (nondimensional; time / temperature / energy scales
    1e-10, 1e3, 1e6)."""
    rng = np.random.default_rng([seed, 4])
    a = rng.integers(0, N_SPECIES, N_REACT)
    b = (a + rng.integers(1, N_SPECIES, N_REACT)) % N_SPECIES
    A = 10.0 ** rng.uniform(8.0, 12.0, N_REACT) * 1e-10
    Ta = rng.uniform(5e3, 2e4, N_REACT) / 1e3
    q = rng.uniform(1e5, 1e6, N_REACT) / 1e6
    return np.stack([a.astype(float), b.astype(float), A, Ta, q])


class ReactingEulerProblem(FomProblem):
    """Configuration-4 reacting Euler model.

    The reference has no reacting model; the model is defined in
    DESIGN.md §9 / oracle/reacting.py: conserved [rho, m, E, rho Y_0..9],
    periodic, Rusanov fluxes as ``SodProblem`` plus 12 first-order Arrhenius
    reactions a_j -> b_j releasing q_j.  Residual, FD Jacobian, implicit
    step, sampled residual and the adaptive-ROM session run on the device.
    """

    n_var = 3 + N_SPECIES
    boundary = "periodic"
    # primitive fields (the keys of primitive_fields, as SodProblem's)
    var_names = ("rho", "v", "p") + tuple(f"Y{k}" for k in range(N_SPECIES))
    kind = REACTING

    def __init__(self, n_elem: int, gamma: float = 1.4, length: float = 1.0, seed: int = 4,
                 n_pulses: int = 1):
        super().__init__(n_elem, length)
        self.n_pulses = int(n_pulses)
        if gamma <= 1.0:
            raise ValueError("gamma must exceed 1")
        self.gamma = float(gamma)
        self.seed = int(seed)
        self.mechanism = reacting_mechanism(seed)
        self._mech_dev = None

    def primitive_fields(self, q):
        """rho, v, p as the Sod model (fom.py:279-282) from the first three
        conserved variables (the FGS feature maps read these) and the mass
        fractions Y_k = (rho Y_k) / rho (diagnostics, driver.py:168-199)."""
        if _dev.is_device(q):
            t = _dev.torch()
            u = q.reshape(self.n_elem, self.n_var)
            rho = t.clamp_min(u[:, 0], PRIM_FLOOR)
            vel = u[:, 1] / rho
            p = t.clamp_min((self.gamma - 1.0) * (u[:, 2] - (0.5 * rho) * (vel * vel)), PRIM_FLOOR)
        else:
            u = np.asarray(q, dtype=float).reshape(self.n_elem, self.n_var)
            rho = np.maximum(u[:, 0], PRIM_FLOOR)
            vel = u[:, 1] / rho
            p = np.maximum((self.gamma - 1.0) * (u[:, 2] - (0.5 * rho) * (vel * vel)), PRIM_FLOOR)
        out = {"rho": rho, "v": vel, "p": p}
        for k in range(N_SPECIES):
            out[f"Y{k}"] = u[:, 3 + k] / rho
        return out

    def abi(self) -> Model:
        if self._mech_dev is None:  # uploaded on first device use
            self._mech_dev = _dev.dev(self.mechanism.ravel().copy())
        return Model(self.kind, self.n_var, self.n_elem, self.dx, 0.0, self.gamma,
                     ptr(self._mech_dev))

    def initial_state(self) -> np.ndarray:
        """BASELINE cfg 4: rho = 1, u = 0, p = 1 plus a seeded sinusoidal
        pressure/temperature pulse (amplitude U[0.5, 1], centre U[0.3, 0.7],
        width 0.1), or n_pulses narrow ones (amplitude U[0.2, 1], centre
        U[0, 1) periodic, width U[0.002, 0.01]); species fractions
        Y_k = (k+1)/55.  Host-generated input data."""
        n = self.n_elem
        x = (np.arange(n) + 0.5) / n
        p = np.ones(n)
        if self.n_pulses == 1:
            rng = np.random.default_rng([self.seed, 5])
            amp, cen, wid = rng.uniform(0.5, 1.0), rng.uniform(0.3, 0.7), 0.1
            d = x - cen
            p = 1.0 + np.where(np.abs(d) < 0.5 * wid,
                               amp * 0.5 * (1.0 + np.cos(2.0 * np.pi * d / wid)), 0.0)
        else:
            rng = np.random.default_rng([self.seed, 6])
            amp = rng.uniform(0.2, 1.0, self.n_pulses)
            cen = rng.uniform(0.0, 1.0, self.n_pulses)
            wid = rng.uniform(0.002, 0.01, self.n_pulses)
            for a, c, w in zip(amp, cen, wid):
                d = np.mod(x - c + 0.5, 1.0) - 0.5
                p = p + np.where(np.abs(d) < 0.5 * w,
                                 a * 0.5 * (1.0 + np.cos(2.0 * np.pi * d / w)), 0.0)
        out = np.zeros((n, self.n_var))
        out[:, 0] = 1.0
        out[:, 2] = p / (self.gamma - 1.0)
        for k in range(N_SPECIES):
            out[:, 3 + k] = 1.0 * ((k + 1) / 55.0)
        return out.ravel()


def _check_model(model):
    if not isinstance(model, (BurgersProblem, SodProblem, ReactingEulerProblem)):
        raise TypeError(
            f"{type(model).__name__} has no device implementation; the B200 path "
            "supports BurgersProblem and SodProblem (subclasses may override "
            "initial_state only)")


def fd_jacobian_blocks(model: FomProblem, q):
    """Nonzero blocks of ``fd_jacobian`` (fom.py:301-328), shape
    (n_elem, 3, n_var, n_var): d rhs_i / d q_{left(i)}, d q_i, d q_{right(i)}."""
    _check_model(model)
    qd = _dev.dev(q)
    nv = model.n_var
    out = _dev.empty(model.n_elem, 3, nv, nv)
    m = model.abi()
    Context.get().call("adrom_fd_jacobian_blocks", C.byref(m), ptr(qd), ptr(out))
    return _dev.like(out, q)


def fd_jacobian(model: FomProblem, q, rhs0=None):
    """Dense FD Jacobian (fom.py:301-328) assembled from the device blocks.
    O(N^2) memory like the reference — for small grids / tests only."""
    blocks = _dev.host(fd_jacobian_blocks(model, q))
    nv, n = model.n_var, model.n_elem
    dense = np.zeros((n * nv, n * nv))
    cells = np.arange(n)
    left, right = model.neighbor_cells(cells)
    for i in range(n):
        rows = slice(i * nv, (i + 1) * nv)
        if left[i] != i:
            dense[rows, left[i] * nv:(left[i] + 1) * nv] = blocks[i, 0]
        dense[rows, i * nv:(i + 1) * nv] = blocks[i, 1]
        if right[i] != i:
            dense[rows, right[i] * nv:(right[i] + 1) * nv] = blocks[i, 2]
    return dense


def implicit_step(model: FomProblem, q, dt: float, stepper: TimeStepper | None = None) -> NewtonResult:
    """fom.py:331-347 — backward Euler by Newton; non-convergence flagged."""
    _check_model(model)
    if stepper is None:
        stepper = TimeStepper(dt=dt)
    if stepper.newton_tol <= 0:
        raise DenseError("newton_solve requires tol > 0")
    qd = _dev.dev(q)
    x = _dev.empty(model.n_dof)
    info = NewtonInfo()
    m = model.abi()
    Context.get().call("adrom_implicit_step", C.byref(m), ptr(qd), C.c_double(dt),
                       C.c_double(stepper.newton_tol), C.c_int32(stepper.newton_max_iter),
                       ptr(x), C.byref(info))
    return NewtonResult(x=_dev.like(x, q), converged=bool(info.converged),
                        iterations=int(info.iterations), residual_norm=float(info.residual_norm))


def coarse_step(model: FomProblem, y, z: int, dt: float,
                stepper: TimeStepper | None = None) -> NewtonResult:
    """fom.py:350-356 — implicit step of size z*dt."""
    if z < 1:
        raise ValueError("z must be at least 1")
    return implicit_step(model, y, z * dt, stepper)
