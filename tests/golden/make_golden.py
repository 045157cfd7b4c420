"""Generate golden fixtures by running the REAL reference package.

Run in the build container (the reference tree is mounted read-only at
/root/reference; it does not exist on the GPU box):

    python tests/golden/make_golden.py

Writes ``tests/golden/*.npz``.  Every array is produced by calling the
reference's own public functions (``adrom`` from /root/reference/pkg/src);
the oracle (``oracle/``) and the CUDA path are both checked against these
files.  Inputs are seeded (numpy default_rng) so the script is
reproducible.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(OUT.parents[1]))

import adrom  # noqa: E402
from adrom import driver, fom, projection, sampling, snapshots, tracking  # noqa: E402
from adrom.dense import thin_svd  # noqa: E402

from paper_2605_28684_b200.configs import burgers_bump_ic  # noqa: E402


def save(name, **arrays):
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print(f"wrote {name}.npz: " + ", ".join(f"{k}{np.shape(v)}" for k, v in arrays.items()))


def residuals():
    out = {}
    cases = []
    m = fom.BurgersProblem(4, nu=0.01)
    cases.append(("burgers", 4, 0.01, np.array([1.0, 0.0, 0.0, 0.0])))
    cases.append(("burgers", 1024, 1e-3, burgers_bump_ic(1024)))
    rng = np.random.default_rng(11)
    cases.append(("burgers", 1027, 0.02, rng.standard_normal(1027)))
    cases.append(("sod", 64, 1.4, fom.sod_initial_state(64)))
    u = np.empty((65, 3))
    u[:, 0] = rng.uniform(0.3, 1.5, 65)
    vel = rng.uniform(-0.8, 0.8, 65)
    p = rng.uniform(0.1, 1.5, 65)
    u[:, 1] = u[:, 0] * vel
    u[:, 2] = p / 0.4 + 0.5 * u[:, 0] * vel ** 2
    cases.append(("sod", 65, 1.4, u.ravel()))
    # a state that trips the density / pressure floors
    v = u.copy()
    v[3, 0] = -1e-3
    v[7, 2] = 0.0
    cases.append(("sod", 65, 1.4, v.ravel()))
    for i, (kind, n, par, q) in enumerate(cases):
        m = fom.BurgersProblem(n, nu=par) if kind == "burgers" else fom.SodProblem(n, gamma=par)
        out[f"q{i}"] = q
        out[f"f{i}"] = m.rhs(q)
        out[f"meta{i}"] = np.array([0 if kind == "burgers" else 1, n, par])
        # gather form at every cell (rhs_at_cells), random cell order
        cells = rng.permutation(n)[: max(4, n // 3)]
        left, right = m.neighbor_cells(cells)
        nv = m.n_var
        g = np.stack([q.reshape(n, nv)[left], q.reshape(n, nv)[cells], q.reshape(n, nv)[right]], axis=1)
        out[f"cells{i}"] = cells
        out[f"fc{i}"] = m.rhs_at_cells(g)
    out["ncases"] = np.array(len(cases))
    save("residuals", **out)


def jacobians():
    out = {}
    i = 0
    for n in (7, 8, 9, 10):
        rng = np.random.default_rng(n)
        m = fom.BurgersProblem(n, nu=0.03)
        q = rng.standard_normal(n)
        out[f"q{i}"], out[f"J{i}"], out[f"meta{i}"] = q, fom.fd_jacobian(m, q), np.array([0, n, 0.03])
        i += 1
    for n in (6, 7, 8):
        m = fom.SodProblem(n)
        q = fom.sod_initial_state(n)
        out[f"q{i}"], out[f"J{i}"], out[f"meta{i}"] = q, fom.fd_jacobian(m, q), np.array([1, n, 1.4])
        i += 1
    m = fom.SodProblem(12)
    rng = np.random.default_rng(5)
    q = fom.sod_initial_state(12) * (1 + 0.05 * rng.standard_normal(36))
    out[f"q{i}"], out[f"J{i}"], out[f"meta{i}"] = q, fom.fd_jacobian(m, q), np.array([1, 12, 1.4])
    i += 1
    out["ncases"] = np.array(i)
    save("jacobians", **out)


def newton():
    out = {}
    cases = [
        (fom.BurgersProblem(64, nu=1e-3), burgers_bump_ic(64), 1e-3),
        (fom.BurgersProblem(1024, nu=1e-3), burgers_bump_ic(1024), 1e-3),
        (fom.BurgersProblem(100, nu=0.01), fom.BurgersProblem(100, nu=0.01).initial_state(), 0.01),
        (fom.SodProblem(64), fom.sod_initial_state(64), 2.5e-4 * 5),
        (fom.SodProblem(200), fom.sod_initial_state(200), 1e-3),
    ]
    for i, (m, q, dt) in enumerate(cases):
        res = fom.implicit_step(m, q, dt)
        kind = 0 if isinstance(m, fom.BurgersProblem) else 1
        par = m.nu if kind == 0 else m.gamma
        out[f"q{i}"] = q
        out[f"x{i}"] = res.x
        out[f"info{i}"] = np.array([res.converged, res.iterations, res.residual_norm])
        out[f"meta{i}"] = np.array([kind, m.n_elem, par, dt])
    # non-convergence flag (test_fom.py:203-207)
    m = fom.BurgersProblem(8, nu=0.01)
    res = fom.implicit_step(m, m.initial_state(), 1.0,
                            fom.TimeStepper(dt=1.0, newton_tol=1e-15, newton_max_iter=1))
    out["nc_q"] = m.initial_state()
    out["nc_x"] = res.x
    out["nc_info"] = np.array([res.converged, res.iterations, res.residual_norm])
    out["ncases"] = np.array(len(cases))
    save("newton", **out)


def isvd():
    out = {}
    rng = np.random.default_rng(2024)
    n, r, k, lam, steps = 300, 8, 12, 0.7, 40
    modes = np.linalg.qr(rng.standard_normal((n, k)))[0]
    spec = np.arange(1, k + 1) ** -1.0
    stream = np.stack([modes @ (spec * rng.standard_normal(k)) + 1e-6 * rng.standard_normal(n)
                       for _ in range(steps + r)])
    res = thin_svd(stream[:r].T)
    basis = tracking.ReducedBasis(phi=res.u[:, :r], sigma=res.s[:r].copy())
    out["stream"], out["phi0"], out["sigma0"] = stream, basis.phi, basis.sigma
    sig_hist = []
    for y in stream[r:]:
        basis = tracking.isvd_update(basis, y, lam, r)
        sig_hist.append(basis.sigma)
    out["phiN"], out["sigma_hist"] = basis.phi, np.array(sig_hist)
    out["meta"] = np.array([n, r, k, lam, steps])
    # known-answer cases (test_tracking.py:36-102)
    b = tracking.ReducedBasis(phi=np.eye(4)[:, :1], sigma=np.array([1.0]))
    o = tracking.isvd_update(b, np.eye(4)[:, 0], lam=1.0, r=1)
    out["ka_inspan_sigma"] = o.sigma
    b = tracking.ReducedBasis(phi=np.eye(5)[:, :2], sigma=np.array([2.0, 1.0]))
    o = tracking.isvd_update(b, np.zeros(5), lam=0.5, r=2)
    out["ka_zero_sigma"], out["ka_zero_phi"] = o.sigma, o.phi
    phi, _ = np.linalg.qr(np.random.default_rng(1).standard_normal((8, 3)))
    b = tracking.ReducedBasis(phi=phi, sigma=np.array([2.0, 1.0, 0.5]))
    y = phi @ np.array([0.3, -0.2, 0.1])
    o = tracking.isvd_update(b, y, lam=0.9, r=3)
    out["ka_deg_phi0"], out["ka_deg_y"], out["ka_deg_phi"], out["ka_deg_sigma"] = phi, y, o.phi, o.sigma
    save("isvd", **out)


def sampling_cases():
    out = {}
    # QDEIM on a Burgers POD basis (cfg-0 physics, small window)
    m = fom.BurgersProblem(512, nu=1e-3)
    states = [burgers_bump_ic(512)]
    for _ in range(80):
        states.append(fom.implicit_step(m, states[-1], 5e-4).x)
    sc = driver._fit_scaling_for(m, np.array(states))
    y = np.column_stack([sc.preprocess(q) for q in states])
    basis = snapshots.pod(y, 8)
    out["pod_y"], out["pod_phi"], out["pod_sigma"] = y, basis.phi, basis.sigma
    s = sampling.qdeim_sample(basis, 8)
    out["q_piv"] = s.indices
    s2 = sampling.qdeim_sample(basis, 20)
    out["q_piv_restart"] = s2.indices
    out["q_pinv"] = sampling.build_deim_operator(basis, s)
    out["q_pinv_restart"] = sampling.build_deim_operator(basis, s2)
    rng = np.random.default_rng(77)
    rnd = np.linalg.qr(rng.standard_normal((400, 6)))[0]
    out["rnd_phi"] = rnd
    out["rnd_piv"] = sampling.qdeim_sample(tracking.ReducedBasis(rnd, np.ones(6)), 6).indices
    # FGS on Sod
    ms = fom.SodProblem(256)
    q = fom.sod_initial_state(256)
    for _ in range(10):
        q = fom.implicit_step(ms, q, 5e-4).x
    phi = np.linalg.qr(rng.standard_normal((768, 6)))[0]
    fmap = sampling.FeatureMap(kind="pressure-gradient", n_extra=30)
    sf = sampling.fgs_sample(tracking.ReducedBasis(phi, np.ones(6)), q, 36, fmap, ms)
    sfc = sampling.stencil_closure(sf, ms)
    out["fgs_q"], out["fgs_phi"], out["fgs_idx"], out["fgs_closure"] = q, phi, sf.indices, sfc.closure
    save("sampling", **out)


def rom_steps():
    out = {}
    m = fom.BurgersProblem(16, nu=0.01)
    states = [m.initial_state()]
    for _ in range(6):
        states.append(fom.implicit_step(m, states[-1], 1e-3).x)
    sc = snapshots.fit_scaling(states, 1)
    y = np.column_stack([sc.preprocess(q) for q in states])
    basis = snapshots.pod(y, 4)
    samp = sampling.stencil_closure(sampling.qdeim_sample(basis, 4), m)
    out["b_phi"], out["b_qref"], out["b_phinorm"] = basis.phi, sc.q_ref, sc.phi_norm
    out["b_idx"], out["b_clo"] = samp.indices, samp.closure
    for kind in ("lspg", "galerkin"):
        op = projection.build_rom_operator(basis, sc, samp, m, kind)
        prev = projection.encode(states[-1], op)
        res = projection.rom_step(op, m, prev, 1e-3)
        out[f"b_a0"] = prev.a
        out[f"b_{kind}_a"] = res.state.a
        out[f"b_{kind}_info"] = np.array([res.converged, res.iterations, res.residual_norm])
        out["b_pinv"] = op.deim_pinv
    # Sod operator with FGS sampling
    ms = fom.SodProblem(64)
    states = [fom.sod_initial_state(64)]
    for _ in range(12):
        states.append(fom.implicit_step(ms, states[-1], 1e-3).x)
    sc = snapshots.fit_scaling(states, 3)
    y = np.column_stack([sc.preprocess(q) for q in states])
    basis = snapshots.pod(y, 6)
    samp = sampling.stencil_closure(
        sampling.fgs_sample(basis, states[-1], 15,
                            sampling.FeatureMap("pressure-gradient", n_extra=9), ms), ms)
    out["s_phi"], out["s_qref"], out["s_phinorm"] = basis.phi, sc.q_ref, sc.phi_norm
    out["s_idx"], out["s_clo"] = samp.indices, samp.closure
    for kind in ("lspg", "galerkin"):
        op = projection.build_rom_operator(basis, sc, samp, ms, kind)
        prev = projection.encode(states[-1], op)
        res = projection.rom_step(op, ms, prev, 1e-3)
        out["s_a0"] = prev.a
        out[f"s_{kind}_a"] = res.state.a
        out[f"s_{kind}_info"] = np.array([res.converged, res.iterations, res.residual_norm])
        out["s_pinv"] = op.deim_pinv
    save("romstep", **out)


class _Recorder:
    """Wraps driver-level reference functions to record the loop's internals."""

    def __init__(self):
        self.sigma, self.steps, self.samplings = [], [], []

    def install(self):
        orig_isvd, orig_step = driver.isvd_update, driver.rom_step
        orig_sampling = driver._build_sampling

        def isvd_rec(basis, y_hat, lam, r):
            out = orig_isvd(basis, y_hat, lam, r)
            self.sigma.append(out.sigma.copy())
            return out

        def step_rec(op, model, state, dt, tol=1e-8, max_iter=10):
            out = orig_step(op, model, state, dt, tol=tol, max_iter=max_iter)
            self.steps.append((out.state.a.copy(), out.iterations, out.converged))
            return out

        def samp_rec(config, model, basis, y_corr):
            out = orig_sampling(config, model, basis, y_corr)
            self.samplings.append(out.indices.copy())
            return out

        driver.isvd_update, driver.rom_step, driver._build_sampling = isvd_rec, step_rec, samp_rec
        return lambda: (setattr(driver, "isvd_update", orig_isvd),
                        setattr(driver, "rom_step", orig_step),
                        setattr(driver, "_build_sampling", orig_sampling))


def run_loop(name, cfg, ic=None):
    if ic is not None:
        class Custom(fom.BurgersProblem):
            def initial_state(self):
                return ic.copy()
        orig = driver.make_problem
        driver.make_problem = lambda c: Custom(c.n_elem, nu=c.nu)
    try:
        truth = driver.run_fom(driver.ExperimentConfig(**{**cfg.__dict__, "mode": "fom"}))
        rec = _Recorder()
        undo = rec.install()
        try:
            res = driver.run_adaptive_rom(cfg, truth=truth.trajectory)
        finally:
            undo()
    finally:
        if ic is not None:
            driver.make_problem = orig
    ev = [{k: (v if not isinstance(v, (np.bool_, bool)) else bool(v)) for k, v in e.items()}
          for e in res.event_log]
    env_state, env_sigma, env_samp = _envelope(cfg, truth.trajectory, res.trajectory,
                                               np.array(rec.sigma), ic, rec.samplings)
    save(name, truth=truth.trajectory, traj=res.trajectory,
         sigma=np.array(rec.sigma), a=np.array([s[0] for s in rec.steps]),
         it=np.array([s[1] for s in rec.steps]), conv=np.array([s[2] for s in rec.steps]),
         samplings=np.array(rec.samplings, dtype=object) if len({len(s) for s in rec.samplings}) > 1
         else np.array(rec.samplings),
         errors=res.errors, events=np.array(json.dumps(ev, default=float)),
         failures=np.array(res.newton_failures, dtype=np.int64),
         env_state=env_state, env_sigma=env_sigma, env_samp_stable=env_samp)


def _envelope(cfg, truth, traj, sigma, ic, samplings, seeds=(1, 2, 3, 4, 5)):
    """The reference's own sensitivity to rounding-level perturbations at the
    places where any other implementation's arithmetic necessarily differs
    from numpy/LAPACK's: every coarse Newton result, every iSVD output
    (basis and singular values), every reduced-step result and every state
    transfer are nudged by one ulp at random entries.
    Records the per-step relative state spread and the per-event sigma
    spread (max over seeds).  Trajectory-level parity gates are expressed
    relative to this envelope: an implementation that differs from the
    reference only in rounding cannot be held to a tighter bound than the
    reference's sensitivity to its own rounding."""
    orig_coarse = driver.coarse_step
    orig_isvd = driver.isvd_update
    orig_step = driver.rom_step
    orig_encode = driver.encode
    if ic is not None:
        class Custom(fom.BurgersProblem):
            def initial_state(self):
                return ic.copy()
        orig_mp = driver.make_problem
        driver.make_problem = lambda c: Custom(c.n_elem, nu=c.nu)
    worst_state = np.zeros(traj.shape[0])
    worst_sigma = np.zeros(sigma.shape)
    stable = np.ones(len(samplings), dtype=bool)  # sampling decision unchanged by the nudges

    def nudge(rng, x):
        mask = rng.random(x.shape) < 0.5
        return np.where(mask, np.nextafter(x, np.inf), x)

    try:
        for seed in seeds:
            rng = np.random.default_rng(seed)

            def nudged(model, y, z, dt, stepper=None):
                res = orig_coarse(model, y, z, dt, stepper)
                res.x = nudge(rng, res.x)
                return res

            def isvd_nudged(basis, y_hat, lam, r):
                out = orig_isvd(basis, y_hat, lam, r)
                return tracking.ReducedBasis(phi=nudge(rng, out.phi), sigma=nudge(rng, out.sigma))

            def step_nudged(op, model, state, dt, tol=1e-8, max_iter=10):
                out = orig_step(op, model, state, dt, tol=tol, max_iter=max_iter)
                st = projection.ReducedState(a=nudge(rng, out.state.a), n=out.state.n)
                return projection.RomStepResult(state=st, converged=out.converged,
                                                iterations=out.iterations,
                                                residual_norm=out.residual_norm)

            def encode_nudged(q, op, n=0):
                out = orig_encode(q, op, n)
                return projection.ReducedState(a=nudge(rng, out.a), n=out.n)

            driver.coarse_step = nudged
            driver.isvd_update = isvd_nudged
            driver.rom_step = step_nudged
            driver.encode = encode_nudged
            rec = _Recorder()
            undo = rec.install()  # records the nudged iSVD outputs
            try:
                out = driver.run_adaptive_rom(cfg, truth=truth)
            finally:
                undo()
                driver.coarse_step = orig_coarse
                driver.isvd_update = orig_isvd
                driver.rom_step = orig_step
                driver.encode = orig_encode
            dev = np.linalg.norm(out.trajectory - traj, axis=1) / np.linalg.norm(traj, axis=1)
            worst_state = np.maximum(worst_state, dev)
            sg = np.array(rec.sigma)
            if sg.shape == sigma.shape:
                worst_sigma = np.maximum(worst_sigma, np.abs(sg / sigma - 1.0))
            for k, (a, b) in enumerate(zip(rec.samplings, samplings)):
                if list(a) != list(b):
                    stable[k] = False
    finally:
        driver.coarse_step = orig_coarse
        driver.isvd_update = orig_isvd
        driver.rom_step = orig_step
        driver.encode = orig_encode
        if ic is not None:
            driver.make_problem = orig_mp
    return worst_state, worst_sigma, stable


def loops():
    U = tracking.UpdateRule
    run_loop("loop_burgers64", driver.ExperimentConfig(
        model="burgers", n_elem=64, nu=0.01, dt=1e-3, n_t=60, r=4, n_s=4, w_init=4, z=10,
        projection="lspg", sampling="qdeim", mode="adaptive", rule=U("isvd", lam=0.1)))
    run_loop("loop_burgers256_bump", driver.ExperimentConfig(
        model="burgers", n_elem=256, nu=1e-3, dt=1e-4, n_t=300, r=8, n_s=8, w_init=150, z=10,
        projection="lspg", sampling="qdeim", mode="adaptive", rule=U("isvd", lam=0.1)),
        ic=burgers_bump_ic(256))
    run_loop("loop_burgers64_galerkin", driver.ExperimentConfig(
        model="burgers", n_elem=64, nu=0.01, dt=1e-3, n_t=60, r=4, n_s=6, w_init=4, z=7,
        projection="galerkin", sampling="qdeim", mode="adaptive", rule=U("isvd", lam=0.5)))
    run_loop("loop_sod64_fgs", driver.ExperimentConfig(
        model="sod", n_elem=64, dt=2.5e-4, n_t=40, r=4, n_s=6, w_init=4, z=10,
        sampling="fgs", feature="pressure-gradient", n_extra=2, rule=U("isvd", lam=0.1)))
    run_loop("loop_sod128_fgs_z5", driver.ExperimentConfig(
        model="sod", n_elem=128, dt=4e-4, n_t=120, r=8, n_s=21, w_init=20, z=5,
        sampling="fgs", feature="pressure-gradient", n_extra=13, rule=U("isvd", lam=0.25)))


def cfg0_loop(n_online=500, stride=10):
    """BASELINE configuration 0 as defined (Burgers N=1024, nu=1e-3, seeded
    bump IC, dt=1e-4, w_init=2000 -> POD of 2001 states, r=n_s=16, z=10,
    lambda=0.1, LSPG + QDEIM) over the first ``n_online`` online steps, run
    by the real reference.  Stored compactly: the offline results the GPU
    run injects (q_ref, basis, q_last), decoded states every ``stride``
    steps, and every per-step / per-event decision."""
    ic = burgers_bump_ic(1024)
    cfg = driver.ExperimentConfig(
        model="burgers", n_elem=1024, nu=1e-3, dt=1e-4, n_t=2000 + n_online, r=16, n_s=16,
        w_init=2000, z=10, projection="lspg", sampling="qdeim", mode="adaptive",
        rule=tracking.UpdateRule("isvd", lam=0.1))

    class Custom(fom.BurgersProblem):
        def initial_state(self):
            return ic.copy()
    orig = driver.make_problem
    driver.make_problem = lambda c: Custom(c.n_elem, nu=c.nu)
    try:
        truth = driver.run_fom(driver.ExperimentConfig(**{**cfg.__dict__, "mode": "fom"}))
        rec = _Recorder()
        undo = rec.install()
        try:
            res = driver.run_adaptive_rom(cfg, truth=truth.trajectory)
        finally:
            undo()
    finally:
        driver.make_problem = orig
    tr = truth.trajectory
    training = tr[: cfg.w_init + 1]
    scaling = snapshots.ScalingTransform(q_ref=training[0].copy(), phi_norm=np.ones(1))
    y_train = np.column_stack([scaling.preprocess(q) for q in training])
    basis0 = snapshots.pod(y_train, cfg.r)
    ev = [{k: (v if not isinstance(v, (np.bool_, bool)) else bool(v)) for k, v in e.items()}
          for e in res.event_log]
    env_state, env_sigma, env_samp = _envelope(cfg, tr, res.trajectory, np.array(rec.sigma), ic,
                                               rec.samplings, seeds=(1, 2, 3))
    keep = np.arange(cfg.w_init + stride, cfg.n_t + 1, stride)
    save("loop_cfg0", q_ref=training[0], q_last=training[-1], phi0=basis0.phi,
         sigma0=basis0.sigma, steps=keep, traj=res.trajectory[keep], truth=tr[keep],
         sigma=np.array(rec.sigma), it=np.array([s[1] for s in rec.steps]),
         conv=np.array([s[2] for s in rec.steps]), samplings=np.array(rec.samplings),
         errors=res.errors, events=np.array(json.dumps(ev, default=float)),
         failures=np.array(res.newton_failures, dtype=np.int64),
         env_state=env_state[keep], env_sigma=env_sigma, env_samp_stable=env_samp,
         wall=np.array(res.wall_seconds), n_online=np.array(n_online))


def io_artifacts():
    """The reference's artifact writers (io.py) on a synthetic Sod RunResult:
    the exact bytes of every file, for the format tests of
    paper_2605_28684_b200.io."""
    import tempfile
    from adrom import io as rio
    rng = np.random.default_rng(5)
    cfg = driver.ExperimentConfig(model="sod", n_elem=16, dt=1e-3, n_t=24, w_init=8, r=4, n_s=6,
                                  z=4, sampling="fgs", n_extra=2,
                                  rule=tracking.UpdateRule("isvd", lam=0.25), save_stride=5,
                                  label="golden-io")
    m = fom.SodProblem(16)
    traj = np.stack([m.initial_state() * (1.0 + 0.01 * k) + 1e-3 * rng.standard_normal(48)
                     for k in range(25)])
    steps = np.arange(9, 25)
    errors = rng.uniform(1e-6, 1e-2, (16, 3))
    sig_steps = np.array([12, 16, 20, 24])
    sig_err = rng.uniform(1e-6, 1e-2, (4, 3))
    res = driver.RunResult(config=cfg, kind="adaptive", trajectory=traj, wall_seconds=0.125,
                           var_names=m.var_names, newton_failures=[11, 17], error_steps=steps,
                           errors=errors, event_log=[{"event": 1, "step": 12, "coarse_converged": True,
                                                      "coarse_iterations": 3,
                                                      "residual_norm": 0.5}],
                           signal_steps=sig_steps, signal_errors=sig_err)
    out = {"traj": traj, "errors": errors, "sig_err": sig_err, "sig_steps": sig_steps}
    with tempfile.TemporaryDirectory() as d:
        run_dir = Path(d) / "run-golden"
        run_dir.mkdir()
        files = {"error_history.csv": rio.write_error_history,
                 "signal_errors.csv": rio.write_signal_errors,
                 "profiles.csv": rio.write_profiles, "snapshots.csv": rio.write_snapshots}
        for name, fn in files.items():
            fn(run_dir / name, res)
            out["file_" + name] = np.array((run_dir / name).read_text())
        rio.write_manifest(run_dir, res, list(files), fom_wall=1.5)
        out["file_manifest.json"] = np.array((run_dir / "manifest.json").read_text())
    out["cache_key"] = np.array(rio.fom_cache_key(cfg))
    out["config_dict"] = np.array(json.dumps(rio.config_to_dict(cfg)))
    save("io_artifacts", **out)


def dense_rules():
    """Known answers of the dense helpers and the five non-iSVD update rules
    (dense.py:75-200, snapshots.py:54-89, tracking.py:67-93, :181-246,
    fom.py:222-236), from the reference's own functions on seeded inputs."""
    from adrom import dense
    rng = np.random.default_rng(2605)
    out = {}
    # least squares: tall full rank, matrix rhs, rank deficient (min norm)
    a = rng.standard_normal((300, 7))
    b = rng.standard_normal(300)
    out["ls_a0"], out["ls_b0"], out["ls_x0"] = a, b, dense.least_squares(a, b)
    bm = rng.standard_normal((300, 5))
    out["ls_a1"], out["ls_b1"], out["ls_x1"] = a, bm, dense.least_squares(a, bm)
    a2 = a.copy()
    a2[:, 3] = 2.0 * a2[:, 1] - a2[:, 5]  # exactly dependent column
    out["ls_a2"], out["ls_b2"], out["ls_x2"] = a2, b, dense.least_squares(a2, b)
    # orth (sign-fixed thin QR)
    a3 = rng.standard_normal((513, 9))
    out["orth_a"], out["orth_q"] = a3, dense.orth(a3)
    # pivoted QR pivots
    a4 = rng.standard_normal((6, 40))
    piv, q, r = dense.pivoted_qr(a4, 5)
    out["pqr_a"], out["pqr_piv"] = a4, piv
    # principal angles
    u = np.linalg.qr(rng.standard_normal((200, 4)))[0]
    v = np.linalg.qr(u + 1e-7 * rng.standard_normal((200, 4)))[0]
    out["pa_u"], out["pa_v"], out["pa_theta"] = u, v, dense.principal_angles(u, v)
    w = np.linalg.qr(rng.standard_normal((200, 3)))[0]
    out["pa_w"], out["pa_theta2"] = w, dense.principal_angles(u, w)
    # newton on a 2-d system
    res_f = lambda x: np.array([x[0] ** 2 + x[1] ** 2 - 4.0, x[0] - x[1]])  # noqa: E731
    jac_f = lambda x: np.array([[2 * x[0], 2 * x[1]], [1.0, -1.0]])  # noqa: E731
    nr = dense.newton_solve(res_f, jac_f, np.array([1.0, 0.5]), 1e-12, 20)
    out["newton_x"], out["newton_it"] = nr.x, np.array(nr.iterations)
    # fit_scaling + pod: tall (Sod window), wide (Burgers), plain pod
    m = fom.SodProblem(96)
    st = [m.initial_state()]
    stepper = fom.TimeStepper(dt=2e-3)
    for _ in range(30):
        st.append(fom.implicit_step(m, st[-1], 2e-3, stepper).x)
    st = np.array(st)
    sc = snapshots.fit_scaling(list(st), 3)
    y = np.column_stack([sc.preprocess(q) for q in st])
    bas = snapshots.pod(y, 6)
    out["pod_train"], out["pod_qref"], out["pod_phinorm"] = st, sc.q_ref, sc.phi_norm
    out["pod_phi"], out["pod_sigma"] = bas.phi, bas.sigma
    yw = rng.standard_normal((40, 70)) @ np.diag(np.logspace(0, -8, 70)) @ rng.standard_normal((70, 90))
    bw = snapshots.pod(yw, 12)
    out["podw_y"], out["podw_phi"], out["podw_sigma"] = yw, bw.phi, bw.sigma
    # rusanov flux on a batch
    ul = np.abs(rng.standard_normal((50, 3))) + np.array([0.2, 0.0, 1.0])
    ur = np.abs(rng.standard_normal((50, 3))) + np.array([0.2, 0.0, 1.0])
    out["rus_ul"], out["rus_ur"], out["rus_f"] = ul, ur, fom.rusanov_flux(ul, ur, 1.4)
    # the rules on one basis / window
    n, r = 400, 5
    phi = np.linalg.qr(rng.standard_normal((n, r)))[0]
    sig = np.linspace(3.0, 1.0, r)
    basis = tracking.ReducedBasis(phi, sig)
    yy = [rng.standard_normal(n) + phi @ rng.standard_normal(r) for _ in range(8)]
    win = tracking.SnapshotWindow(6, initial=yy[:7])
    win.push(yy[7])
    out["rule_phi"], out["rule_sig"], out["rule_win"] = phi, sig, win.matrix
    out["rule_y"], out["rule_a"] = yy[7], rng.standard_normal(r)
    out["wsvd_phi"] = tracking.wsvd_update(win, r).phi
    out["wsvd_sig"] = tracking.wsvd_update(win, r).sigma
    out["direct_phi"] = tracking.direct_update(basis, win).phi
    out["onestep_phi"] = tracking.onestep_update(basis, yy[7], out["rule_a"]).phi
    out["oja_phi"] = tracking.oja_update(basis, yy[7], 0.05).phi
    out["grouse_phi"] = tracking.grouse_update(basis, yy[7], 0.05).phi
    save("dense_rules", **out)


def rule_loops():
    """The adaptive loop with each non-iSVD rule and the every-step cadence
    (driver.py:276-288, :346-387), real reference runs on small grids."""
    U = tracking.UpdateRule
    base = dict(model="burgers", n_elem=96, nu=0.01, dt=1e-3, n_t=70, r=4, n_s=6, w_init=10, z=5,
                projection="lspg", sampling="qdeim", mode="adaptive")
    cases = {
        "rule_wsvd": dict(rule=U("wsvd", window=6)),
        "rule_direct": dict(rule=U("direct", window=8)),
        "rule_onestep": dict(rule=U("onestep")),
        "rule_oja": dict(rule=U("oja", eta=0.05)),
        "rule_grouse": dict(rule=U("grouse", eta=0.05)),
        "rule_isvd_everystep": dict(rule=U("isvd", lam=0.5), cadence="every-step"),
        "rule_oja_everystep_sod": dict(model="sod", n_elem=64, dt=5e-4, n_t=50, w_init=8, r=4, n_s=8,
                                       sampling="fgs", n_extra=4, rule=U("oja", eta=0.02),
                                       cadence="every-step"),
    }
    out = {}
    for name, kw in cases.items():
        cfg = driver.ExperimentConfig(**{**base, **kw})
        truth = driver.run_fom(driver.ExperimentConfig(**{**cfg.__dict__, "mode": "fom"}))
        res = driver.run_adaptive_rom(cfg, truth=truth.trajectory)
        ev = [{k: (v if not isinstance(v, (np.bool_, bool)) else bool(v)) for k, v in e.items()}
              for e in res.event_log]
        out[name + "_cfg"] = np.array(json.dumps({k: (v.__dict__ if hasattr(v, "__dict__") else v)
                                                  for k, v in {**base, **kw}.items()}))
        out[name + "_truth"] = truth.trajectory
        out[name + "_traj"] = res.trajectory
        out[name + "_errors"] = res.errors
        out[name + "_sig_errors"] = res.signal_errors
        out[name + "_events"] = np.array(json.dumps(ev, default=float))
    save("rule_loops", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["residuals", "jacobians", "newton", "isvd", "sampling_cases",
                             "rom_steps", "loops"]
    for w in which:
        globals()[w]()
    (OUT / "PROVENANCE.json").write_text(json.dumps({
        "generator": "tests/golden/make_golden.py",
        "reference": str(REF), "adrom_version": adrom.__version__,
        "numpy": np.__version__,
    }, indent=1) + "\n")
