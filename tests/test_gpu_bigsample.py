"""Large sampled sets (csrc/bigsample.cu): grid-wide FGS ranking, closure /
gather plan, CholeskyQR2 DEIM pseudo-inverse and the multi-kernel LSPG
Gauss-Newton step that configuration 4 (408,954 sampled rows) needs.

The one-block path and the grid-wide path implement the same reference
functions (sampling.py:117-189, projection.py:158-204); ADROM_BIG_SAMPLES=1
/ ADROM_FGS_GRID=1 force the grid-wide path at small sizes so it is checked
against the same golden vectors and oracle loops as the one-block path.
"""

import numpy as np
import pytest

from oracle import hyper, online, physics, reacting as R, subspace

pytestmark = pytest.mark.gpu


def _pkg():
    import paper_2605_28684_b200 as P
    return P


@pytest.fixture
def grid_path(monkeypatch):
    monkeypatch.setenv("ADROM_BIG_SAMPLES", "1")
    monkeypatch.setenv("ADROM_FGS_GRID", "1")


@pytest.mark.parametrize("n_cells,n_s,n_extra", [(9000, 400, 380), (20000, 3000, 2990)])
def test_fgs_grid_ranking_vs_oracle(n_cells, n_s, n_extra):
    """> 8192 cells: the radix-sort ranking (sampling.py:117-159), rows equal."""
    P = _pkg()
    m = physics.Model("sod", n_cells)
    x = (np.arange(n_cells) + 0.5) / n_cells
    rng = np.random.default_rng(7)
    rho = 1.0 + 0.3 * np.tanh((x - 0.3) / 0.01) + 0.01 * rng.standard_normal(n_cells)
    p = 1.0 + 0.5 * np.tanh((x - 0.6) / 0.02)
    p[100:110] = p[99]  # ties -> lowest cell first
    q = np.stack([rho, 0.1 * rho, p / 0.4 + 0.5 * rho * 0.01], axis=1).ravel()
    phi = np.linalg.qr(rng.standard_normal((3 * n_cells, 20)))[0]
    want = hyper.fgs(phi, q, n_s, n_extra, "pressure-gradient", m, exact_greedy=True)
    got = P.fgs_sample(P.ReducedBasis(phi=phi, sigma=np.ones(20)), q, n_s,
                       P.FeatureMap("pressure-gradient", n_extra), P.SodProblem(n_cells))
    assert list(got.indices) == list(want.indices)


LOOP = dict(n=128, dt=2e-3, n_t=60, w_init=20, r=8, n_cells=3, z=5, lam=0.25)


def test_reacting_loop_grid_path_vs_oracle(grid_path):
    P = _pkg()
    L = LOOP
    n, n_extra = L["n"], L["n_cells"] * 13
    n_s = L["r"] + n_extra
    m = physics.Model("reacting", n, gamma=1.4, mech=tuple(R.mechanism().ravel()))
    ocfg = online.LoopConfig(model=m, dt=L["dt"], n_t=L["n_t"], w_init=L["w_init"], r=L["r"],
                             n_s=n_s, n_extra=n_extra, z=L["z"], lam=L["lam"], sampling="fgs")
    training = online.training_states(ocfg, R.initial_state(n))
    q_ref, phi_norm = subspace.fit_scaling(list(training), 13)
    _, d, phi0, sigma0 = online.offline(ocfg, training)
    rec = online.run_online(ocfg, training, q_ref, d, phi0, sigma0)
    cfg = P.ExperimentConfig(model="reacting", n_elem=n, dt=L["dt"], n_t=L["n_t"],
                             w_init=L["w_init"], r=L["r"], n_s=n_s, n_extra=n_extra, z=L["z"],
                             sampling="fgs", rule=P.UpdateRule("isvd", lam=L["lam"]))
    res = P.run_adaptive_rom(cfg, truth=training, offline=(
        P.ScalingTransform(q_ref=q_ref, phi_norm=phi_norm), P.ReducedBasis(phi0, sigma0)))
    got = res.trajectory[cfg.w_init + 1:]
    want = np.array(rec.states)
    dev = np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)
    assert dev.max() < 1e-8, dev.max()
    assert len(res.event_log) == len(rec.events)
    assert all("update_error" not in e for e in res.event_log)
    assert res.newton_failures == rec.failures


@pytest.mark.parametrize("name", ["loop_sod128_fgs_z5", "loop_burgers64"])
def test_golden_loops_grid_path(golden, grid_path, name):
    """The reference's own trajectories (tests/golden) through the grid path."""
    import test_gpu_rom as T
    P = _pkg()
    g = golden(name)
    cfg = T._exp_config(name)
    res = P.run_adaptive_rom(cfg, truth=g["truth"], offline=T._oracle_offline(name, g))
    traj = g["traj"][cfg.w_init + 1:]
    got = res.trajectory[cfg.w_init + 1:]
    dev = np.linalg.norm(got - traj, axis=1) / np.linalg.norm(traj, axis=1)
    env = g["env_state"][cfg.w_init + 1:]
    assert np.all(dev <= np.maximum(1e-9, 10.0 * env)), (dev.max(), env.max())
    it_ref = np.array([int(x) for x in g["it"]])
    diff = np.abs(it_ref - np.asarray(res.step_iterations))
    loose = env > 1e-9
    assert np.all(diff[~loose] == 0) and np.all(diff <= 1), np.flatnonzero(diff)


def test_cfg1_grid_path_matches_one_block_path(monkeypatch):
    """Configuration 1 (Sod 4096 cells, FGS 615 rows) takes the grid-wide
    reduced operator by default (n_s >= 256); it must reproduce the one-block
    path's trajectory (same offline stage, same events)."""
    P = _pkg()
    from paper_2605_28684_b200 import configs
    case = configs.cfg1()
    cfg = P.ExperimentConfig(model="sod", n_elem=case.n_elem, dt=case.dt,
                             n_t=case.w_init + 25, w_init=case.w_init, r=case.r, n_s=case.n_s,
                             z=case.z, sampling="fgs", n_extra=case.n_extra,
                             rule=P.UpdateRule("isvd", lam=case.lam))
    runs = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("ADROM_BIG_SAMPLES", flag)
        runs[flag] = P.run_adaptive_rom(cfg)
    a, b = runs["0"].trajectory, runs["1"].trajectory
    dev = np.linalg.norm(a - b, axis=1) / np.linalg.norm(a, axis=1)
    assert dev.max() < 1e-9, dev.max()
    assert [e["coarse_iterations"] for e in runs["0"].event_log] == \
        [e["coarse_iterations"] for e in runs["1"].event_log]
    assert list(runs["0"].step_iterations) == list(runs["1"].step_iterations)
