"""Pin the CPU oracle against golden vectors produced by the real reference
(tests/golden/make_golden.py) and against the reference tests' known answers.

These run without a GPU.  The oracle is the checker for every GPU parity
test, so it must itself reproduce the reference first.
"""

import json

import numpy as np
import pytest

from oracle import hyper, online, physics, reduced, subspace
from paper_2605_28684_b200.configs import burgers_bump_ic


def _model(meta):
    kind, n, par = int(meta[0]), int(meta[1]), float(meta[2])
    if kind == 0:
        return physics.Model("burgers", n, nu=par)
    return physics.Model("sod", n, gamma=par)


# ---------------------------------------------------------------- residuals

def test_residuals_bitwise(golden):
    g = golden("residuals")
    for i in range(int(g["ncases"])):
        m = _model(g[f"meta{i}"])
        q = g[f"q{i}"]
        assert np.array_equal(physics.rhs(m, q), g[f"f{i}"]), i
        cells = g[f"cells{i}"]
        lft, rgt = m.neighbours(cells)
        qc = q.reshape(m.n_elem, m.n_var)
        st = np.stack([qc[lft], qc[cells], qc[rgt]], axis=1)
        assert np.array_equal(physics.rhs_from_stencils(m, st), g[f"fc{i}"]), i


def test_burgers_hand_stencil():
    # tests/test_fom.py:52-59
    m = physics.Model("burgers", 4, nu=0.01)
    f = physics.rhs(m, np.array([1.0, 0.0, 0.0, 0.0]))
    assert np.allclose(f, [-4.32, 0.16, 0.0, 0.16], atol=1e-14)


def test_rusanov_hand_value():
    # tests/test_fom.py:79-90
    s = np.sqrt(1.4)
    got = physics.rusanov(np.array([1.0, 0.0, 2.5]), np.array([0.125, 0.0, 0.25]), 1.4)
    assert np.allclose(got, [0.5 * s * 0.875, 0.55, 0.5 * s * 2.25], atol=1e-14)


def test_sampled_evaluate_equals_full_rhs():
    # SamplingPlan.evaluate over all rows == rhs, bitwise
    for m, q in ((physics.Model("burgers", 1027, nu=0.01), burgers_bump_ic(1027)),
                 (physics.Model("sod", 515), physics.sod_state(515) *
                  (1 + 0.01 * np.sin(np.arange(515 * 3))))):
        s = hyper.closure(hyper.Sampling(np.arange(m.n_dof), np.arange(m.n_dof)), m)
        plan = hyper.gather_plan(m, s)
        assert np.array_equal(plan.evaluate(m, q[s.closure]), physics.rhs(m, q))


# ---------------------------------------------------------------- Jacobian / Newton

def test_fd_jacobian_blocks_equal_reference_dense(golden):
    g = golden("jacobians")
    for i in range(int(g["ncases"])):
        m = _model(g[f"meta{i}"])
        blocks = physics.fd_jacobian_blocks(m, g[f"q{i}"])
        assert np.array_equal(physics.blocks_to_dense(m, blocks), g[f"J{i}"]), i


def test_implicit_step_matches_reference(golden):
    g = golden("newton")
    for i in range(int(g["ncases"])):
        meta = g[f"meta{i}"]
        m = _model(meta[:3])
        res = physics.implicit_step(m, g[f"q{i}"], float(meta[3]))
        conv, iters, _ = g[f"info{i}"]
        assert res.converged == bool(conv) and res.iterations == int(iters), i
        x_ref = g[f"x{i}"]
        assert np.linalg.norm(res.x - x_ref) <= 1e-13 * np.linalg.norm(x_ref), i


def test_newton_nonconvergence_flag(golden):
    g = golden("newton")
    m = physics.Model("burgers", 8, nu=0.01)
    res = physics.implicit_step(m, g["nc_q"], 1.0, tol=1e-15, max_iter=1)
    assert not res.converged and res.iterations == 1
    assert np.allclose(res.x, g["nc_x"], rtol=1e-13)


# ---------------------------------------------------------------- iSVD

def test_isvd_stream_matches_reference(golden):
    g = golden("isvd")
    n, r, k, lam, steps = g["meta"]
    r = int(r)
    phi, sigma = g["phi0"], g["sigma0"]
    for j, y in enumerate(g["stream"][r:]):
        phi, sigma, _ = subspace.isvd_update(phi, sigma, y, float(lam), r)
        assert np.allclose(sigma, g["sigma_hist"][j], rtol=1e-12, atol=0), j
    assert subspace.principal_angles(phi, g["phiN"]).max() < 1e-12


def test_isvd_known_answers(golden):
    g = golden("isvd")
    phi, s, _ = subspace.isvd_update(np.eye(4)[:, :1], np.array([1.0]), np.eye(4)[:, 0], 1.0, 1)
    assert np.allclose(s, [np.sqrt(2.0)]) and np.allclose(s, g["ka_inspan_sigma"])
    phi, s, _ = subspace.isvd_update(np.eye(5)[:, :2], np.array([2.0, 1.0]), np.zeros(5), 0.5, 2)
    assert np.allclose(s, [1.0, 0.5]) and np.allclose(s, g["ka_zero_sigma"])
    phi, s, info = subspace.isvd_update(g["ka_deg_phi0"], np.array([2.0, 1.0, 0.5]),
                                        g["ka_deg_y"], 0.9, 3)
    assert info["degenerate"]
    assert subspace.principal_angles(phi, g["ka_deg_phi"]).max() <= 1e-12
    assert np.allclose(s, g["ka_deg_sigma"], rtol=1e-13)


# ---------------------------------------------------------------- sampling / operator

def test_qdeim_matches_reference(golden):
    g = golden("sampling")
    phi = g["pod_phi"]
    assert list(hyper.qdeim(phi, 8).indices) == list(g["q_piv"])
    assert list(hyper.qdeim(phi, 8, exact_greedy=True).indices) == list(g["q_piv"])
    assert list(hyper.qdeim(phi, 20).indices) == list(g["q_piv_restart"])
    assert list(hyper.qdeim(phi, 20, exact_greedy=True).indices) == list(g["q_piv_restart"])
    assert list(hyper.qdeim(g["rnd_phi"], 6, exact_greedy=True).indices) == list(g["rnd_piv"])
    assert np.allclose(hyper.deim_pinv(phi, g["q_piv"]), g["q_pinv"], rtol=1e-10, atol=1e-12)
    assert np.allclose(hyper.deim_pinv(phi, g["q_piv_restart"]), g["q_pinv_restart"],
                       rtol=1e-10, atol=1e-12)


def test_pod_matches_reference(golden):
    g = golden("sampling")
    phi, sigma = subspace.pod(g["pod_y"], 8)
    assert np.allclose(sigma, g["pod_sigma"], rtol=1e-12)
    assert np.allclose(phi, g["pod_phi"], atol=1e-12)


def test_fgs_matches_reference(golden):
    g = golden("sampling")
    m = physics.Model("sod", 256)
    s = hyper.fgs(g["fgs_phi"], g["fgs_q"], 36, 30, "pressure-gradient", m)
    assert list(s.indices) == list(g["fgs_idx"])
    assert list(hyper.closure(s, m).closure) == list(g["fgs_closure"])


@pytest.mark.parametrize("tag,kind,n", [("b", "burgers", 16), ("s", "sod", 64)])
def test_rom_steps_match_reference(golden, tag, kind, n):
    g = golden("romstep")
    m = physics.Model(kind, n, nu=0.01)
    d = subspace.row_scale(g[f"{tag}_phinorm"], n)
    samp = hyper.Sampling(g[f"{tag}_idx"], g[f"{tag}_clo"])
    op = reduced.build_operator(m, g[f"{tag}_phi"], g[f"{tag}_qref"], d, samp)
    assert np.allclose(op.pinv, g[f"{tag}_pinv"], rtol=1e-11, atol=1e-13)
    a0 = g[f"{tag}_a0"]
    for name, fn in (("lspg", reduced.lspg_step), ("galerkin", reduced.galerkin_step)):
        out = fn(op, m, a0, 1e-3)
        conv, iters, _ = g[f"{tag}_{name}_info"]
        assert out.converged == bool(conv) and out.iterations == int(iters)
        assert np.allclose(out.a, g[f"{tag}_{name}_a"], rtol=1e-10, atol=1e-12)


# ---------------------------------------------------------------- online loop

LOOPS = {
    "loop_burgers64": dict(model=physics.Model("burgers", 64, nu=0.01), dt=1e-3, n_t=60,
                           w_init=4, r=4, n_s=4, z=10, lam=0.1),
    "loop_burgers256_bump": dict(model=physics.Model("burgers", 256, nu=1e-3), dt=1e-4, n_t=300,
                                 w_init=150, r=8, n_s=8, z=10, lam=0.1),
    "loop_burgers64_galerkin": dict(model=physics.Model("burgers", 64, nu=0.01), dt=1e-3,
                                    n_t=60, w_init=4, r=4, n_s=6, z=7, lam=0.5,
                                    projection="galerkin"),
    "loop_sod64_fgs": dict(model=physics.Model("sod", 64), dt=2.5e-4, n_t=40, w_init=4, r=4,
                           n_s=6, z=10, lam=0.1, sampling="fgs", n_extra=2),
    "loop_sod128_fgs_z5": dict(model=physics.Model("sod", 128), dt=4e-4, n_t=120, w_init=20,
                               r=8, n_s=21, z=5, lam=0.25, sampling="fgs", n_extra=13),
}


@pytest.mark.parametrize("name", sorted(LOOPS))
def test_online_loop_matches_reference(golden, name):
    g = golden(name)
    cfg = online.LoopConfig(**LOOPS[name])
    truth = g["truth"]
    training = truth[: cfg.w_init + 1]
    q_ref, d, phi0, sigma0 = online.offline(cfg, training)
    rec = online.run_online(cfg, training, q_ref, d, phi0, sigma0)
    traj = g["traj"][cfg.w_init + 1:]
    got = np.array(rec.states)
    # per-step relative state error, gated by the reference's own 1-ulp
    # sensitivity envelope (make_golden._envelope); 1e-9 floor
    dev = np.linalg.norm(got - traj, axis=1) / np.linalg.norm(traj, axis=1)
    env = g["env_state"][cfg.w_init + 1:]
    assert np.all(dev <= np.maximum(1e-9, 10.0 * env)), (dev.max(), env.max())
    ref = g["sigma"]
    err = np.abs(np.array(rec.sigma) - ref)
    tol = np.maximum(1e-8 * ref + 1e-12 * ref[:, :1], 10.0 * g["env_sigma"] * ref)
    assert np.all(err <= tol)
    events = json.loads(str(g["events"]))
    assert len(events) == len(rec.events)
    for j, (e_ref, e) in enumerate(zip(events, rec.events)):
        # the residual norm ||y - Phi Phi^T y|| is a cancellation: a basis
        # perturbation of relative size e moves it by ~e ||y||.  Gate it by the
        # reference's own sigma envelope at the previous event times ||y||
        # (finite, so a gross mismatch still fails)
        prior = float(g["env_sigma"][j - 1].max()) if j > 0 else 0.0
        y_hat = d * (rec.signal[j + 1][1] - q_ref)
        atol = 10.0 * prior * float(np.linalg.norm(y_hat)) + 1e-14
        assert e_ref["coarse_iterations"] == e["coarse_iterations"]
        assert e_ref["coarse_converged"] == e["coarse_converged"]
        assert "update_error" not in e_ref and "update_error" not in e
        assert abs(e_ref["residual_norm"] - e["residual_norm"]) <= 1e-8 * e_ref["residual_norm"] + atol
    samp_ref = [list(s) for s in g["samplings"]]
    assert samp_ref == [list(s) for s in rec.samplings]
