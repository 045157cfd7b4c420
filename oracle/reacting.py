"""Oracle: residual of the configuration-4 reacting Euler model.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

PARITY UNPINNED.  The reference has no reacting model at all (SPEC.md:8,
SURVEY.md §8a row a3: "no reference code ... numpy oracle (builder-defined)").
This module *is* the definition of the model; the CUDA kernel
is checked against it, and both against the conservation identities below.

Model (nondimensional, periodic, n_var = 13, layout q[cell*13 + var]; the
initial state follows BASELINE.json configs[4]):

  U = [rho, m, E, rho Y_0 .. rho Y_9]
  primitives as the Sod model (fom.py:204-210): rho = max(U0, 1e-10),
    u = m / rho, p = max((gamma - 1)(E - 0.5 rho u^2), 1e-10), T = p / rho
  flux F = [m, m u + p, u (E + p), m Y_k]  with Y_k = U_{3+k} / rho
  interfaces: Rusanov (fom.py:222-236) with s = max(|u| + sqrt(gamma p / rho))
  sources: 12 irreversible first-order reactions  a_j -> b_j,
    w_j = A_j exp(-Ta_j / T) max(U_{3+a_j}, 0)
    S_{3+a_j} -= w_j,  S_{3+b_j} += w_j,  S_E += q_j w_j
  R_i = -(F_{i+1/2} - F_{i-1/2}) / dx + S(U_i)

Mechanism (seeded, SURVEY §8d cfg 4): A_j = 10**U[8, 12] * 1e-10 (time scale
1e-10), Ta_j = U[5e3, 2e4] / 1e3 (temperature scale 1e3), q_j = U[1e5, 1e6] / 1e6
(energy scale 1e6), a_j uniform in 0..9, b_j = (a_j + U{1..9}) mod 10.

Conservation identities used by the tests: sum_i R_rho = 0, sum_i R_m = 0 and
sum_i sum_k R_{rho Y_k} = 0 up to rounding (periodic flux differences cancel,
reactions move mass between species); with A = 0 a uniform state is an
equilibrium.
"""

from __future__ import annotations

import numpy as np

N_SPECIES = 10
N_REACT = 12
N_VAR = 3 + N_SPECIES
PRIM_FLOOR = 1e-10


def mechanism(seed: int = 4) -> np.ndarray:
    """(5, 12) array: rows a, b (as floats), A, Ta, q."""
    rng = np.random.default_rng([seed, 4])
    a = rng.integers(0, N_SPECIES, N_REACT)
    b = (a + rng.integers(1, N_SPECIES, N_REACT)) % N_SPECIES
    A = 10.0 ** rng.uniform(8.0, 12.0, N_REACT) * 1e-10
    Ta = rng.uniform(5e3, 2e4, N_REACT) / 1e3
    q = rng.uniform(1e5, 1e6, N_REACT) / 1e6
    return np.stack([a.astype(float), b.astype(float), A, Ta, q])


def initial_state(n_elem: int, gamma: float = 1.4, seed: int = 4, n_pulses: int = 1) -> np.ndarray:
    """BASELINE cfg 4: base state rho = 1, p = 1, u = 0 with a seeded sinusoidal
    pressure (hence temperature, T = p/rho) pulse
    p = 1 + a (1 + cos(2 pi (x - c) / w)) / 2 for |x - c| < w/2, a ~ U[0.5, 1],
    c ~ U[0.3, 0.7], w = 0.1; species fractions Y_k = (k+1)/55.

    n_pulses > 1 (the configuration-4 workload, configs.cfg4): that many
    such pulses, a ~ U[0.2, 1], c ~ U[0, 1) (periodic distance),
    w ~ U[0.002, 0.01], drawn from default_rng([seed, 6]) — narrow waves whose
    transport gives the training window more than r = 128 significant POD
    modes (one wide pulse gives ~25-45)."""
    x = (np.arange(n_elem) + 0.5) / n_elem
    p = np.ones(n_elem)
    if n_pulses == 1:
        rng = np.random.default_rng([seed, 5])
        amp, cen, wid = rng.uniform(0.5, 1.0), rng.uniform(0.3, 0.7), 0.1
        d = x - cen
        p = 1.0 + np.where(np.abs(d) < 0.5 * wid, amp * 0.5 * (1.0 + np.cos(2.0 * np.pi * d / wid)), 0.0)
    else:
        rng = np.random.default_rng([seed, 6])
        amp = rng.uniform(0.2, 1.0, n_pulses)
        cen = rng.uniform(0.0, 1.0, n_pulses)
        wid = rng.uniform(0.002, 0.01, n_pulses)
        for a, c, w in zip(amp, cen, wid):
            d = np.mod(x - c + 0.5, 1.0) - 0.5
            p = p + np.where(np.abs(d) < 0.5 * w, a * 0.5 * (1.0 + np.cos(2.0 * np.pi * d / w)), 0.0)
    rho = np.ones(n_elem)
    out = np.zeros((n_elem, N_VAR))
    out[:, 0] = rho
    out[:, 2] = p / (gamma - 1.0)
    for k in range(N_SPECIES):
        out[:, 3 + k] = rho * ((k + 1) / 55.0)
    return out.ravel()


def _prims(c, gamma):
    rho = np.maximum(c[..., 0], PRIM_FLOOR)
    vel = c[..., 1] / rho
    kin = (0.5 * rho) * (vel * vel)
    p = np.maximum((gamma - 1.0) * (c[..., 2] - kin), PRIM_FLOOR)
    return rho, vel, p


def _flux(c, gamma):
    rho, vel, p = _prims(c, gamma)
    out = np.empty_like(c)
    out[..., 0] = c[..., 1]
    out[..., 1] = c[..., 1] * vel + p
    out[..., 2] = vel * (c[..., 2] + p)
    for k in range(N_SPECIES):
        out[..., 3 + k] = c[..., 1] * (c[..., 3 + k] / rho)
    return out


def rusanov(left, right, gamma):
    rl, vl, pl = _prims(left, gamma)
    rr, vr, pr = _prims(right, gamma)
    speed = np.maximum(np.abs(vl) + np.sqrt(gamma * pl / rl), np.abs(vr) + np.sqrt(gamma * pr / rr))
    avg = 0.5 * (_flux(left, gamma) + _flux(right, gamma))
    return avg - (0.5 * speed)[..., None] * (right - left)


def sources(c, gamma, mech):
    rho, _, p = _prims(c, gamma)
    temp = p / rho
    s = np.zeros_like(c)
    for j in range(N_REACT):
        a, b = int(mech[0, j]), int(mech[1, j])
        w = (mech[2, j] * np.exp(-mech[3, j] / temp)) * np.maximum(c[..., 3 + a], 0.0)
        s[..., 3 + a] -= w
        s[..., 3 + b] += w
        s[..., 2] += mech[4, j] * w
    return s


def rhs(q, n_elem, dx, gamma, mech):
    """Full residual, periodic grid."""
    cells = np.asarray(q, dtype=float).reshape(n_elem, N_VAR)
    right = np.roll(cells, -1, axis=0)
    face = rusanov(cells, right, gamma)          # face i = i+1/2
    lo = np.roll(face, 1, axis=0)                 # i-1/2
    div = -(face - lo) / dx
    return (div + sources(cells, gamma, mech)).ravel()
