"""Oracle: the online loop of the history-aware iSVD adaptive ROM.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Restates ``/root/reference/pkg/src/adrom/driver.py:291-410`` (``_run_rom``)
for the iSVD rule with every-event cadence (the north-star path), plus the
offline stage it consumes (``driver.py:232-261`` and ``snapshots.py``).
Differences from the reference, all outside the arithmetic:

* the trajectory is kept every ``keep_stride`` steps instead of as a dense
  (n_t+1) x N array (``driver.py:306``; 277 GB at BASELINE config 3);
* the coarse Newton uses the banded restatement of ``oracle.physics``;
* per-event singular values and per-step reduced coordinates are recorded
  so the GPU loop can be compared step by step.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import hyper, physics, reduced, subspace


@dataclass
class LoopConfig:
    """The ``ExperimentConfig`` fields the online loop reads (driver.py:63-91)."""

    model: physics.Model
    dt: float
    n_t: int
    w_init: int
    r: int
    n_s: int
    z: int = 10
    lam: float = 0.1
    projection: str = "lspg"
    sampling: str = "qdeim"
    feature: str = "pressure-gradient"
    n_extra: int = 0
    newton_tol: float = 1e-8
    newton_max_iter: int = 10
    adaptive: bool = True
    isvd_projection: str = "lstsq"
    exact_greedy: bool = False


@dataclass
class LoopRecord:
    steps: list = field(default_factory=list)        # saved step indices
    states: list = field(default_factory=list)       # decoded q~ at saved steps
    reduced: list = field(default_factory=list)      # a after each ROM step (before any transfer)
    sigma: list = field(default_factory=list)        # sigma after each event
    events: list = field(default_factory=list)       # dicts like driver.py:351-387
    samplings: list = field(default_factory=list)    # sampled indices per rebuild
    failures: list = field(default_factory=list)     # rom non-convergence steps
    iterations: list = field(default_factory=list)   # Gauss-Newton iterations per step
    signal: list = field(default_factory=list)       # (step, y_corr) coarse snapshots
    phi_final: np.ndarray | None = None
    a_init: np.ndarray | None = None
    checkpoints: dict = field(default_factory=dict)  # step -> (phi, sigma, q~) after its event


def training_states(cfg: LoopConfig, q0):
    """driver.py:250-261 — q^0 .. q^{w_init} by fine implicit steps."""
    states = [np.asarray(q0, dtype=float)]
    for _ in range(cfg.w_init):
        states.append(physics.implicit_step(cfg.model, states[-1], cfg.dt,
                                            cfg.newton_tol, cfg.newton_max_iter).x)
    return np.array(states)


def offline(cfg: LoopConfig, training):
    """driver.py:296-299 — scaling, preprocessed training matrix, POD."""
    q_ref, phi_norm = subspace.fit_scaling(list(training), cfg.model.n_var)
    d = subspace.row_scale(phi_norm, cfg.model.n_elem)
    y_train = np.column_stack([d * (q - q_ref) for q in training])
    phi0, sigma0 = subspace.pod(y_train, cfg.r)
    return q_ref, d, phi0, sigma0


def _sampling(cfg: LoopConfig, phi, y_corr, pinned=None):
    """driver.py:264-273.  ``pinned``: use these rows instead (the pinned-
    decisions mode of the parity harness)."""
    if pinned is not None:
        idx = np.asarray(pinned, dtype=np.int64)
        return hyper.closure(hyper.Sampling(indices=idx, closure=np.unique(idx)), cfg.model)
    if cfg.sampling == "fgs":
        if y_corr is None:
            raise ValueError("feature-guided sampling needs a correction state")
        s = hyper.fgs(phi, y_corr, cfg.n_s, cfg.n_extra, cfg.feature, cfg.model,
                      exact_greedy=cfg.exact_greedy)
    else:
        s = hyper.qdeim(phi, cfg.n_s, exact_greedy=cfg.exact_greedy)
    return hyper.closure(s, cfg.model)


_NUDGE_ULPS = [1.0]


def _nudge(rng, x):
    """Rounding-level perturbation of random entries (the sensitivity
    envelope): one ulp by default; ``nudge_ulps`` > 1 perturbs every entry by
    a uniform random relative amount of up to that many ulps — the size of
    the rounding differences a different summation order leaves in a length-N
    reduction (~sqrt(N) ulps)."""
    if rng is None:
        return x
    x = np.asarray(x, dtype=float)
    k = _NUDGE_ULPS[0]
    if k <= 1.0:
        return np.where(rng.random(x.shape) < 0.5, np.nextafter(x, np.inf), x)
    return x * (1.0 + k * 2.220446049250313e-16 * rng.uniform(-1.0, 1.0, x.shape))


def _nudge_sigma(rng, s):
    """Singular values: LAPACK's SVD (gesdd) guarantees them only to
    eps ||K|| ABSOLUTE accuracy (backward stability), so the envelope perturbs
    each by up to ``nudge_ulps`` x eps x sigma_1 (the relative one-ulp nudge
    of ``_nudge`` with one ulp)."""
    if rng is None:
        return s
    s = np.asarray(s, dtype=float)
    k = _NUDGE_ULPS[0]
    if k <= 1.0:
        return _nudge(rng, s)
    return s + k * 2.220446049250313e-16 * s[0] * rng.uniform(-1.0, 1.0, s.shape)


def run_online(cfg: LoopConfig, training, q_ref, d, phi0, sigma0, keep_stride=1,
               n_steps=None, nudge_seed=None, pinned_samplings=None,
               checkpoint_steps=(), nudge_ulps=1.0) -> LoopRecord:
    """driver.py:304-390 (one timing pass).  ``n_steps`` truncates the
    horizon to a prefix (for full-size prefix parity).

    ``nudge_seed`` perturbs every coarse Newton result, iSVD output, reduced
    step result and state transfer by one ulp at random entries — the places
    where any other implementation's arithmetic necessarily differs from
    numpy/LAPACK's — to measure the loop's own rounding sensitivity (the
    envelope the parity gates are expressed in; like
    ``tests/golden/make_golden._envelope`` on the reference itself).

    ``pinned_samplings`` (one row set per sampling rebuild, start first)
    replaces the QDEIM/FGS decisions — to compare two loops whose discrete
    decisions are unstable under rounding (configuration 3)."""
    pins = list(pinned_samplings) if pinned_samplings is not None else None
    rng = None if nudge_seed is None else np.random.default_rng(nudge_seed)
    _NUDGE_ULPS[0] = float(nudge_ulps)
    model = cfg.model
    rec = LoopRecord()
    phi, sigma = np.array(phi0, dtype=float), np.array(sigma0, dtype=float)
    q_last = np.asarray(training[cfg.w_init], dtype=float)
    needs_signal = cfg.adaptive or cfg.sampling == "fgs"
    y_corr = None
    if needs_signal:                                     # driver.py:323-327
        res = physics.coarse_step(model, q_last, cfg.z, cfg.dt, cfg.newton_tol,
                                  cfg.newton_max_iter)
        y_corr = res.x
        rec.signal.append((cfg.w_init + cfg.z, y_corr.copy()))
    samp = _sampling(cfg, phi, y_corr, pins[0] if pins else None)  # driver.py:329-331
    rec.samplings.append(samp.indices.copy())
    op = reduced.build_operator(model, phi, q_ref, d, samp)
    a = reduced.encode(op, q_last)
    rec.a_init = a.copy()
    step_fn = reduced.lspg_step if cfg.projection == "lspg" else reduced.galerkin_step
    last = cfg.n_t if n_steps is None else min(cfg.n_t, cfg.w_init + n_steps)
    for n in range(cfg.w_init, last):                    # driver.py:337
        out = step_fn(op, model, a, cfg.dt, cfg.newton_tol, cfg.newton_max_iter)
        if not out.converged:
            rec.failures.append(n + 1)
        rec.iterations.append(int(out.iterations))
        a = _nudge(rng, out.a)
        q_tilde = reduced.decode(op, a)
        rec.reduced.append(a.copy())
        if (n + 1 - cfg.w_init) % keep_stride == 0 or n + 1 == last:
            rec.steps.append(n + 1)
            rec.states.append(q_tilde.copy())
        if not (cfg.adaptive and (n + 1 - cfg.w_init) % cfg.z == 0):
            continue
        event = {"event": len(rec.events) + 1, "step": n + 1}
        try:                                             # driver.py:353-385
            res = physics.coarse_step(model, y_corr, cfg.z, cfg.dt, cfg.newton_tol,
                                      cfg.newton_max_iter)
            y_corr = _nudge(rng, res.x)
            rec.signal.append((n + 1 + cfg.z, y_corr.copy()))
            event["coarse_converged"] = res.converged
            event["coarse_iterations"] = res.iterations
            y_hat = d * (y_corr - q_ref)
            phi_new, sigma_new, _ = subspace.isvd_update(phi, sigma, y_hat, cfg.lam, cfg.r,
                                                         projection=cfg.isvd_projection)
            phi_new, sigma_new = _nudge(rng, phi_new), _nudge_sigma(rng, sigma_new)
            event["residual_norm"] = float(np.linalg.norm(y_hat - phi @ (phi.T @ y_hat)))
            samp_new = _sampling(cfg, phi_new, y_corr,
                                 pins[len(rec.samplings)] if pins else None)
            op = reduced.build_operator(model, phi_new, q_ref, d, samp_new)
            phi, sigma = phi_new, sigma_new
            rec.samplings.append(samp_new.indices.copy())
            a = _nudge(rng, reduced.encode(op, q_tilde))
            event["a_transfer"] = a.copy()
            if n + 1 in checkpoint_steps:
                rec.checkpoints[n + 1] = (phi.copy(), sigma.copy(), q_tilde.copy())
        except Exception as exc:  # noqa: BLE001 — driver.py:384-385
            event["update_error"] = f"{type(exc).__name__}: {exc}"
        rec.sigma.append(sigma.copy())
        rec.events.append(event)
    rec.phi_final = phi
    return rec
