"""Configuration-4 model inside the adaptive-ROM loop (SURVEY §8a rows a3,
a5, a9-a12 for the reacting Euler model).

The reference has no reacting model: parity is against the
oracle (oracle/reacting.py defines the model; oracle/online.py restates
driver.py:291-410).  Sampled residuals are bitwise; the loop uses the same
gates as the Burgers / Sod loops (trajectory 1e-8 relative, FGS rows and
iteration counts equal, sigma 1e-8).
"""

import numpy as np
import pytest

from oracle import hyper, online, physics, reacting as R, subspace

pytestmark = pytest.mark.gpu


def _pkg():
    import paper_2605_28684_b200 as P
    return P


def _model(n):
    return physics.Model("reacting", n, gamma=1.4, mech=tuple(R.mechanism().ravel()))


def test_sampled_residual_bitwise():
    P = _pkg()
    n = 64
    m = _model(n)
    rng = np.random.default_rng(3)
    q = R.initial_state(n) * (1.0 + 0.01 * rng.standard_normal(n * 13))
    idx = rng.choice(n * 13, 40, replace=False)
    s = hyper.closure(hyper.Sampling(indices=idx, closure=None), m)
    want = hyper.gather_plan(m, s).evaluate(m, q[s.closure])
    pm = P.ReactingEulerProblem(n)
    samp = P.stencil_closure(P.SamplingSet(indices=idx, closure=np.unique(idx)), pm)
    plan = P.SamplingPlan(pm, samp)
    got = plan.evaluate(q[samp.closure])
    assert np.array_equal(got, want)
    # rhs_at_cells on gathered stencils (fom.py:190-198 semantics)
    cells = np.unique(idx // 13)
    st = np.stack([q.reshape(n, 13)[(cells - 1) % n], q.reshape(n, 13)[cells],
                   q.reshape(n, 13)[(cells + 1) % n]], axis=1)
    assert np.array_equal(pm.rhs_at_cells(st), physics.rhs_from_stencils(m, st))


LOOP = dict(n=128, dt=2e-3, n_t=60, w_init=20, r=8, n_cells=3, z=5, lam=0.25)


@pytest.mark.parametrize("projection", ["lspg", "galerkin"])
def test_reacting_adaptive_loop_vs_oracle(projection):
    P = _pkg()
    L = LOOP
    n, n_extra = L["n"], L["n_cells"] * 13
    n_s = L["r"] + n_extra
    m = _model(n)
    ocfg = online.LoopConfig(model=m, dt=L["dt"], n_t=L["n_t"], w_init=L["w_init"], r=L["r"],
                             n_s=n_s, n_extra=n_extra, z=L["z"], lam=L["lam"], sampling="fgs",
                             projection=projection)
    training = online.training_states(ocfg, R.initial_state(n))
    q_ref, phi_norm = subspace.fit_scaling(list(training), 13)
    _, d, phi0, sigma0 = online.offline(ocfg, training)
    rec = online.run_online(ocfg, training, q_ref, d, phi0, sigma0)
    cfg = P.ExperimentConfig(model="reacting", n_elem=n, dt=L["dt"], n_t=L["n_t"],
                             w_init=L["w_init"], r=L["r"], n_s=n_s, n_extra=n_extra, z=L["z"],
                             sampling="fgs", projection=projection,
                             rule=P.UpdateRule("isvd", lam=L["lam"]))
    res = P.run_adaptive_rom(cfg, truth=training, offline=(
        P.ScalingTransform(q_ref=q_ref, phi_norm=phi_norm), P.ReducedBasis(phi0, sigma0)))
    got = res.trajectory[cfg.w_init + 1:]
    want = np.array(rec.states)
    dev = np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)
    assert dev.max() < 1e-8, dev.max()
    assert len(res.event_log) == len(rec.events)
    for e_ref, e in zip(rec.events, res.event_log):
        assert "update_error" not in e
        assert e_ref["coarse_iterations"] == e["coarse_iterations"]
    assert res.newton_failures == rec.failures


def test_reacting_session_events_vs_oracle():
    """Event by event: FGS rows equal and singular values within 1e-8."""
    P = _pkg()
    from paper_2605_28684_b200.driver import Session, offline_stage
    L = LOOP
    n, n_extra = L["n"], L["n_cells"] * 13
    n_s = L["r"] + n_extra
    m = _model(n)
    ocfg = online.LoopConfig(model=m, dt=L["dt"], n_t=L["n_t"], w_init=L["w_init"], r=L["r"],
                             n_s=n_s, n_extra=n_extra, z=L["z"], lam=L["lam"], sampling="fgs")
    training = online.training_states(ocfg, R.initial_state(n))
    q_ref, phi_norm = subspace.fit_scaling(list(training), 13)
    _, d, phi0, sigma0 = online.offline(ocfg, training)
    rec = online.run_online(ocfg, training, q_ref, d, phi0, sigma0)
    cfg = P.ExperimentConfig(model="reacting", n_elem=n, dt=L["dt"], n_t=L["n_t"],
                             w_init=L["w_init"], r=L["r"], n_s=n_s, n_extra=n_extra, z=L["z"],
                             sampling="fgs", rule=P.UpdateRule("isvd", lam=L["lam"]))
    model = P.make_problem(cfg)
    tr_dev, _, _ = offline_stage(cfg, model, training)
    sess = Session(cfg, model, adaptive=True)
    sess.load(P.ScalingTransform(q_ref=q_ref, phi_norm=phi_norm), P.ReducedBasis(phi0, sigma0),
              tr_dev[cfg.w_init])
    sess.start()
    assert list(sess.sampling().cpu().numpy()) == list(rec.samplings[0])
    for ev in range(cfg.n_events):
        sess.advance(cfg.z)
        _, _, _, sig, _ = sess.read(1, 1)
        ref = rec.sigma[ev]
        err = np.abs(sig.cpu().numpy() - ref)
        assert np.all(err <= 1e-8 * ref + 1e-10 * ref[0]), (ev, (err / ref).max())
        assert list(sess.sampling().cpu().numpy()) == list(rec.samplings[ev + 1]), ev
    sess.close()


@pytest.mark.parametrize("grid_path", [False, True])
def test_cfg4_recipe_scaled_vs_oracle(monkeypatch, grid_path):
    """Configuration 4's recipe (configs.cfg4: seeded narrow pulses, FGS on 3 %
    of the cells on top of r QDEIM rows, z = 20, lambda = 0.25) on 256 cells
    (8 pulses, r = 12, dt = 5e-4: a well-conditioned reduced problem — the
    LSPG Jacobian's condition number stays below 1e3 and every Gauss-Newton
    solve converges), through the one-block and the grid-wide (bigsample.cu,
    the full-size path) reduced operator."""
    import math
    if grid_path:
        monkeypatch.setenv("ADROM_BIG_SAMPLES", "1")
        monkeypatch.setenv("ADROM_FGS_GRID", "1")
    P = _pkg()
    n, r = 256, 12
    n_s = math.ceil(0.03 * n) * 13
    dt = 5e-4
    m = _model(n)
    ocfg = online.LoopConfig(model=m, dt=dt, n_t=40 + 60, w_init=40, r=r, n_s=n_s,
                             n_extra=n_s - r, z=20, lam=0.25, sampling="fgs")
    training = online.training_states(ocfg, R.initial_state(n, n_pulses=8))
    q_ref, phi_norm = subspace.fit_scaling(list(training), 13)
    _, d, phi0, sigma0 = online.offline(ocfg, training)
    rec = online.run_online(ocfg, training, q_ref, d, phi0, sigma0)
    cfg = P.ExperimentConfig(model="reacting", n_elem=n, dt=dt, n_t=ocfg.n_t, w_init=40, r=r,
                             n_s=n_s, n_extra=n_s - r, z=20, sampling="fgs",
                             rule=P.UpdateRule("isvd", lam=0.25))
    res = P.run_adaptive_rom(cfg, truth=training, offline=(
        P.ScalingTransform(q_ref=q_ref, phi_norm=phi_norm), P.ReducedBasis(phi0, sigma0)))
    got = res.trajectory[cfg.w_init + 1:]
    want = np.array(rec.states)
    dev = np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)
    assert dev.max() < 1e-8, dev.max()
    assert len(res.event_log) == len(rec.events)
    for e_ref, e in zip(rec.events, res.event_log):
        assert "update_error" not in e
        assert e_ref["coarse_iterations"] == e["coarse_iterations"]
    assert res.newton_failures == rec.failures


def test_reacting_error_history_with_full_truth():
    """driver.py:168-199 on the reacting model: with a truth trajectory over
    the whole horizon the run records per-variable errors (rho, v, p, Y_k)
    at the error steps, and run_fom's device trajectory is that truth."""
    P = _pkg()
    n = 64
    cfg = P.ExperimentConfig(model="reacting", n_elem=n, dt=2e-3, n_t=30, w_init=10, r=6, n_s=6 + 13,
                             n_extra=13, z=5, sampling="fgs", rule=P.UpdateRule("isvd", lam=0.25))
    fom = P.run_fom(cfg)
    m = _model(n)
    ocfg = online.LoopConfig(model=m, dt=cfg.dt, n_t=cfg.n_t, w_init=cfg.w_init, r=cfg.r,
                             n_s=cfg.n_s, n_extra=cfg.n_extra, z=cfg.z, lam=0.25, sampling="fgs")
    truth = online.training_states(ocfg.__class__(**{**ocfg.__dict__, "w_init": cfg.n_t}),
                                   R.initial_state(n))
    dev = np.linalg.norm(np.asarray(fom.trajectory) - truth) / np.linalg.norm(truth)
    assert dev < 1e-12, dev
    res = P.run_adaptive_rom(cfg, truth=truth)
    assert res.errors is not None and res.errors.shape[1] == len(res.var_names) == 13
    assert np.all(np.isfinite(res.errors))
