"""Dense helpers, offline stage and the five non-iSVD update rules on the
device vs the REAL reference's outputs (tests/golden/make_golden.py
dense_rules / rule_loops): least_squares / orth / pivoted_qr /
principal_angles / newton_solve (dense.py:75-171), fit_scaling / pod
(snapshots.py:54-89), rusanov_flux (fom.py:222-236), wsvd / direct /
onestep / oja / grouse (tracking.py:181-246) and the adaptive loop with
each rule and with the every-step cadence (driver.py:276-288, :346-387)."""

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g(golden):
    return golden("dense_rules")


def _h(x):
    from paper_2605_28684_b200 import _dev
    return _dev.host(x)


def test_least_squares(g):
    from paper_2605_28684_b200.dense import least_squares
    for i in range(3):
        x = least_squares(g[f"ls_a{i}"], g[f"ls_b{i}"])
        want = g[f"ls_x{i}"]
        assert np.allclose(x, want, rtol=1e-11, atol=1e-13 * np.abs(want).max()), i


def test_least_squares_errors():
    from paper_2605_28684_b200 import DenseError
    from paper_2605_28684_b200.dense import least_squares
    with pytest.raises(DenseError):
        least_squares(np.ones((3, 5)), np.ones(3))   # wide (dense.py:108)
    bad = np.ones((10, 2))
    bad[3, 1] = np.nan
    with pytest.raises(DenseError):
        least_squares(bad, np.ones(10))


def test_orth_and_pivoted_qr(g):
    from paper_2605_28684_b200.dense import orth, pivoted_qr
    q = orth(g["orth_a"])
    assert np.max(np.abs(q - g["orth_q"])) < 1e-13
    piv, qq, rr = pivoted_qr(g["pqr_a"], 5)
    assert np.array_equal(piv, g["pqr_piv"])
    a = g["pqr_a"]
    assert np.allclose(qq.T @ qq, np.eye(qq.shape[1]), atol=1e-13)
    assert np.allclose(qq @ rr[:, :5], a[:, piv], atol=1e-12)
    d = np.abs(np.diag(rr))
    assert np.all(d[:-1] >= d[1:] * (1 - 1e-12)) and np.allclose(np.tril(rr, -1), 0.0)


def test_principal_angles(g):
    from paper_2605_28684_b200.dense import principal_angles
    th = principal_angles(g["pa_u"], g["pa_v"])
    assert np.allclose(th, g["pa_theta"], rtol=1e-6, atol=1e-15)
    th2 = principal_angles(g["pa_u"], g["pa_w"])
    assert np.allclose(th2, g["pa_theta2"], rtol=1e-10)


def test_newton_solve(g):
    from paper_2605_28684_b200.dense import newton_solve
    res_f = lambda x: np.array([x[0] ** 2 + x[1] ** 2 - 4.0, x[0] - x[1]])  # noqa: E731
    jac_f = lambda x: np.array([[2 * x[0], 2 * x[1]], [1.0, -1.0]])  # noqa: E731
    nr = newton_solve(res_f, jac_f, np.array([1.0, 0.5]), 1e-12, 20)
    assert nr.converged and nr.iterations == int(g["newton_it"])
    assert np.allclose(nr.x, g["newton_x"], rtol=1e-14)


def test_newton_singular_raises():
    from paper_2605_28684_b200 import DenseError
    from paper_2605_28684_b200.dense import newton_solve
    with pytest.raises(DenseError, match="singular Jacobian"):
        newton_solve(lambda x: x + 1.0, lambda x: np.zeros((2, 2)), np.zeros(2), 1e-10, 5)


def test_lu_solve_large():
    import torch
    from paper_2605_28684_b200._lib import Context, ptr
    import ctypes as C
    rng = np.random.default_rng(5)
    n = 700
    a = rng.standard_normal((n, n)) + n ** 0.5 * np.eye(n)
    b = rng.standard_normal(n)
    ad = torch.tensor(a, device="cuda")
    bd = torch.tensor(b, device="cuda")
    Context.get().call("adrom_lu_solve", ptr(ad), C.c_int64(n), ptr(bd))
    x = bd.cpu().numpy()
    assert np.linalg.norm(a @ x - b) <= 1e-12 * np.linalg.norm(a) * np.linalg.norm(x)


def test_fit_scaling_and_pod(g):
    from paper_2605_28684_b200.snapshots import fit_scaling, pod, pod_window
    tr = g["pod_train"]
    sc = fit_scaling(list(tr), 3)
    assert np.array_equal(sc.q_ref, g["pod_qref"])
    assert np.allclose(sc.phi_norm, g["pod_phinorm"], rtol=1e-14)
    y = np.column_stack([sc.preprocess(q) for q in tr])
    b = pod(y, 6)
    assert np.allclose(b.sigma, g["pod_sigma"], rtol=1e-11)
    assert np.max(np.abs(b.phi - g["pod_phi"])) < 1e-10
    bw = pod_window(tr, sc, 6)
    assert np.allclose(_h(bw.sigma), g["pod_sigma"], rtol=1e-11)
    assert np.max(np.abs(_h(bw.phi) - g["pod_phi"])) < 1e-10


def test_pod_wide_rank_deficient(g):
    """Wide window (40 x 90, singular values spanning 1e-8): QR of Y^T and
    the Jacobi SVD of R^T; rank check raises beyond the numerical rank."""
    from paper_2605_28684_b200 import DenseError
    from paper_2605_28684_b200.snapshots import pod
    b = pod(g["podw_y"], 12)
    s = g["podw_sigma"]
    assert np.allclose(b.sigma, s, rtol=1e-9)
    # well-separated leading modes agree elementwise (signs fixed)
    gap = s[:-1] / s[1:]
    k = 6
    assert np.all(gap[:k] > 1.01)
    assert np.max(np.abs(b.phi[:, :k] - g["podw_phi"][:, :k])) < 1e-8
    rank_def = np.outer(np.arange(1, 51.0), np.ones(8)) + 0.0
    with pytest.raises(DenseError, match="numerical rank"):
        pod(rank_def, 3)


def test_pod_large_tall_vs_numpy():
    """Householder path at scale: 2^20 x 65 (the configuration-3 window
    shape at 1/16 of the grid) against numpy's SVD."""
    from paper_2605_28684_b200.snapshots import pod
    import torch
    rng = np.random.default_rng(65)
    n, m = 1 << 20, 65
    y = rng.standard_normal((n, 12)) @ (np.logspace(0, -10, 12)[:, None] * rng.standard_normal((12, m)))
    y += 1e-13 * rng.standard_normal((n, m))
    b = pod(torch.tensor(y, device="cuda"), 10)
    u, s, _ = np.linalg.svd(y, full_matrices=False)
    sig = b.sigma.cpu().numpy()
    assert np.allclose(sig, s[:10], rtol=1e-9)
    from oracle import subspace
    assert subspace.max_angle(u[:, :6], b.phi.cpu().numpy()[:, :6]) < 1e-9


def test_rusanov_flux(g):
    from paper_2605_28684_b200.fom import rusanov_flux
    assert np.array_equal(rusanov_flux(g["rus_ul"], g["rus_ur"], 1.4), g["rus_f"])
    one = rusanov_flux(g["rus_ul"][0], g["rus_ur"][0], 1.4)
    assert np.array_equal(one, g["rus_f"][0])


def test_update_rules(g):
    import paper_2605_28684_b200 as P
    from paper_2605_28684_b200 import tracking as T
    basis = P.ReducedBasis(g["rule_phi"], g["rule_sig"])
    win = T.SnapshotWindow(6, initial=list(g["rule_win"].T))
    assert len(win) == 6
    w = T.wsvd_update(win, 5)
    assert np.max(np.abs(_h(w.phi) - g["wsvd_phi"])) < 1e-10
    assert np.allclose(_h(w.sigma), g["wsvd_sig"], rtol=1e-12)
    d = T.direct_update(basis, win)
    assert np.max(np.abs(_h(d.phi) - g["direct_phi"])) < 1e-10
    o = T.onestep_update(basis, g["rule_y"], g["rule_a"])
    assert np.max(np.abs(_h(o.phi) - g["onestep_phi"])) < 1e-11
    j = T.oja_update(basis, g["rule_y"], 0.05)
    assert np.max(np.abs(_h(j.phi) - g["oja_phi"])) < 1e-11
    gr = T.grouse_update(basis, g["rule_y"], 0.05)
    assert np.max(np.abs(_h(gr.phi) - g["grouse_phi"])) < 1e-11
    # skips (tracking.py:211-212, :238-239)
    assert T.onestep_update(basis, g["rule_y"], np.zeros(5)) is basis
    assert T.grouse_update(basis, np.zeros(400), 0.05) is basis


LOOPS = ["rule_wsvd", "rule_direct", "rule_onestep", "rule_oja", "rule_grouse",
         "rule_isvd_everystep", "rule_oja_everystep_sod"]


@pytest.mark.parametrize("name", LOOPS)
def test_rule_loops_vs_reference(golden, name):
    import paper_2605_28684_b200 as P
    L = golden("rule_loops")
    kw = json.loads(str(L[name + "_cfg"]))
    rule = kw.pop("rule")
    cfg = P.ExperimentConfig(**kw, rule=P.UpdateRule(**rule))
    res = P.run_adaptive_rom(cfg, truth=L[name + "_truth"])
    want = L[name + "_traj"]
    dev = np.linalg.norm(res.trajectory - want, axis=1) / np.linalg.norm(want, axis=1)
    assert dev.max() < 1e-8, (dev.max(), int(dev.argmax()))
    assert np.allclose(res.errors, L[name + "_errors"], rtol=1e-6, atol=1e-12)
    assert np.allclose(res.signal_errors, L[name + "_sig_errors"], rtol=1e-6, atol=1e-12)
    ev_ref = json.loads(str(L[name + "_events"]))
    assert len(res.event_log) == len(ev_ref)
    for a, b in zip(res.event_log, ev_ref):
        assert ("update_error" in a) == ("update_error" in b)
        assert a.get("coarse_iterations") == b.get("coarse_iterations")
        assert np.isclose(a["residual_norm"], b["residual_norm"], rtol=1e-6, atol=1e-11)


def test_operator_with_superset_closure():
    """projection.py:73-79 takes sampling.closure verbatim: a caller closure
    larger than the stencil closure changes the operator's closure arrays
    (shape, sample_pos) but nothing it computes."""
    import paper_2605_28684_b200 as P
    rng = np.random.default_rng(9)
    n = 64
    m = P.BurgersProblem(n, nu=0.01)
    phi = np.linalg.qr(rng.standard_normal((n, 4)))[0]
    basis = P.ReducedBasis(phi, np.ones(4))
    sc = P.ScalingTransform(q_ref=m.initial_state(), phi_norm=np.ones(1))
    s0 = P.stencil_closure(P.SamplingSet(indices=np.array([5, 20, 33, 50]),
                                         closure=np.array([5, 20, 33, 50])), m)
    big = P.SamplingSet(indices=s0.indices, closure=np.unique(np.concatenate([s0.closure, [0, 1, 63]])))
    op0 = P.build_rom_operator(basis, sc, s0, m, "lspg")
    op1 = P.build_rom_operator(basis, sc, big, m, "lspg")
    assert np.array_equal(op1.closure, big.closure)
    assert np.array_equal(op1.closure[op1.sample_pos], big.indices)
    a = rng.standard_normal(4)
    d1 = np.asarray(op1.decode_closure(a))
    d0 = np.asarray(op0.decode_closure(a))
    pos = np.searchsorted(op1.closure, op0.closure)
    assert np.allclose(d1[pos], d0, rtol=1e-13, atol=1e-15)
    st = P.ReducedState(a=a, n=0)
    r0 = P.rom_step(op0, m, st, 1e-3)
    r1 = P.rom_step(op1, m, st, 1e-3)
    assert np.array_equal(np.asarray(r0.state.a), np.asarray(r1.state.a))
