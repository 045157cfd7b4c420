"""GPU parity of the core kernels against the golden vectors (produced by the
real reference) and against the CPU oracle at larger sizes.

Tolerances (BASELINE.json north_star): FOM residuals bitwise (relative 1e-12
is the stated bar; we require equality); FD Jacobian entries bitwise;
Newton iterates 1e-12 relative with equal iteration counts; singular values
relative 1e-8 (here 1e-10 on well-conditioned streams) and basis by largest
principal angle < 1e-8 rad.
"""

import numpy as np
import pytest

from oracle import physics, subspace

pytestmark = pytest.mark.gpu


def _pkg():
    import paper_2605_28684_b200 as P
    return P


def _model(meta):
    P = _pkg()
    kind, n, par = int(meta[0]), int(meta[1]), float(meta[2])
    if kind == 0:
        return P.BurgersProblem(n, nu=par), physics.Model("burgers", n, nu=par)
    return P.SodProblem(n, gamma=par), physics.Model("sod", n, gamma=par)


# ------------------------------------------------------------------ kernel 1

def test_rhs_bitwise_golden(golden):
    g = golden("residuals")
    for i in range(int(g["ncases"])):
        m, _ = _model(g[f"meta{i}"])
        f = m.rhs(g[f"q{i}"])
        assert np.array_equal(f, g[f"f{i}"]), i


def test_rhs_at_cells_bitwise_golden(golden):
    g = golden("residuals")
    for i in range(int(g["ncases"])):
        m, _ = _model(g[f"meta{i}"])
        q = g[f"q{i}"].reshape(m.n_elem, m.n_var)
        cells = g[f"cells{i}"]
        lft, rgt = m.neighbor_cells(cells)
        st = np.stack([q[lft], q[cells], q[rgt]], axis=1)
        assert np.array_equal(m.rhs_at_cells(st), g[f"fc{i}"]), i


@pytest.mark.parametrize("n", [4, 5, 1023, 1024, 1025, 3 * 1024 + 7, 1 << 22])
def test_burgers_rhs_bitwise_vs_oracle(n):
    P = _pkg()
    rng = np.random.default_rng(n)
    q = 1.0 + 0.5 * rng.standard_normal(n)
    q[::7] *= -1.0  # both upwind branches
    m = P.BurgersProblem(n, nu=1e-3)
    assert np.array_equal(m.rhs(q), physics.rhs(physics.Model("burgers", n, nu=1e-3), q))


@pytest.mark.parametrize("n", [4, 255, 256, 257, 4096, 1 << 20])
def test_sod_rhs_bitwise_vs_oracle(n):
    P = _pkg()
    rng = np.random.default_rng(n)
    q = physics.sod_state(n) * (1.0 + 0.05 * rng.standard_normal(3 * n))
    m = P.SodProblem(n)
    assert np.array_equal(m.rhs(q), physics.rhs(physics.Model("sod", n), q))


def test_rhs_device_tensor_roundtrip():
    import torch
    P = _pkg()
    m = P.BurgersProblem(4096, nu=1e-3)
    q = torch.linspace(-1, 1, 4096, dtype=torch.float64, device="cuda")
    f = m.rhs(q)
    assert f.is_cuda
    assert np.array_equal(f.cpu().numpy(), physics.rhs(physics.Model("burgers", 4096, nu=1e-3),
                                                       q.cpu().numpy()))


def test_rhs_rejects_wrong_length():
    P = _pkg()
    with pytest.raises(ValueError):
        P.BurgersProblem(16).rhs(np.zeros(15))


# ------------------------------------------------------------------ Jacobian / Newton

def test_fd_jacobian_bitwise_golden(golden):
    P = _pkg()
    g = golden("jacobians")
    for i in range(int(g["ncases"])):
        m, _ = _model(g[f"meta{i}"])
        assert np.array_equal(P.fd_jacobian(m, g[f"q{i}"]), g[f"J{i}"]), i


@pytest.mark.parametrize("kind,n", [("burgers", 4097), ("burgers", 4098), ("sod", 2049)])
def test_fd_jacobian_blocks_bitwise_vs_oracle(kind, n):
    P = _pkg()
    rng = np.random.default_rng(1)
    if kind == "burgers":
        q = 1.0 + 0.3 * rng.standard_normal(n)
        m, om = P.BurgersProblem(n, nu=1e-3), physics.Model("burgers", n, nu=1e-3)
    else:
        q = physics.sod_state(n) * (1.0 + 0.05 * rng.standard_normal(3 * n))
        m, om = P.SodProblem(n), physics.Model("sod", n)
    got = P.fd_jacobian_blocks(m, q)
    ref = physics.fd_jacobian_blocks(om, q)
    assert np.array_equal(got, ref)


def test_implicit_step_golden(golden):
    P = _pkg()
    g = golden("newton")
    for i in range(int(g["ncases"])):
        meta = g[f"meta{i}"]
        m, _ = _model(meta[:3])
        res = P.implicit_step(m, g[f"q{i}"], float(meta[3]))
        conv, iters, _ = g[f"info{i}"]
        assert res.converged == bool(conv), i
        assert res.iterations == int(iters), i
        x_ref = g[f"x{i}"]
        assert np.linalg.norm(res.x - x_ref) <= 1e-12 * np.linalg.norm(x_ref), i


def test_newton_nonconvergence_flagged(golden):
    P = _pkg()
    g = golden("newton")
    m = P.BurgersProblem(8, nu=0.01)
    res = P.implicit_step(m, g["nc_q"], 1.0, P.TimeStepper(dt=1.0, newton_tol=1e-15,
                                                          newton_max_iter=1))
    assert not res.converged and res.iterations == 1
    assert np.allclose(res.x, g["nc_x"], rtol=1e-12)


@pytest.mark.parametrize("kind,n,dt", [("burgers", 1 << 20, 2e-6), ("burgers", 65537, 1e-4),
                                       ("sod", 4096, 5.2e-4), ("sod", 1 << 16, 2e-5)])
def test_implicit_step_vs_oracle_large(kind, n, dt):
    P = _pkg()
    from paper_2605_28684_b200.configs import burgers_bump_ic
    if kind == "burgers":
        q = burgers_bump_ic(n)
        m, om = P.BurgersProblem(n, nu=1e-3), physics.Model("burgers", n, nu=1e-3)
    else:
        q = physics.sod_state(n)
        m, om = P.SodProblem(n), physics.Model("sod", n)
    res = P.implicit_step(m, q, dt)
    ref = physics.implicit_step(om, q, dt)
    assert res.converged == ref.converged and res.iterations == ref.iterations
    assert np.linalg.norm(res.x - ref.x) <= 1e-12 * np.linalg.norm(ref.x)


def test_fixed_points():
    # tests/test_fom.py:171-185 — constant / uniform states are equilibria
    P = _pkg()
    m = P.BurgersProblem(16, nu=0.01)
    q = np.full(16, 0.7)
    for dt in (1e-3, 0.05, 1.0):
        res = P.implicit_step(m, q, dt)
        assert res.converged and np.max(np.abs(res.x - q)) <= 1e-12
    ms = P.SodProblem(16)
    qs = np.tile(np.array([1.0, 0.25, 2.0]), 16)
    res = P.implicit_step(ms, qs, 1e-3)
    assert res.converged and np.max(np.abs(res.x - qs)) <= 1e-12


def test_coarse_step_z1_equals_fine_step():
    # tests/test_fom.py:211-216 (bitwise)
    P = _pkg()
    m = P.BurgersProblem(64, nu=0.02)
    q = m.initial_state()
    a = P.coarse_step(m, q, 1, 1e-3)
    b = P.implicit_step(m, q, 1e-3)
    assert np.array_equal(a.x, b.x)


# ------------------------------------------------------------------ kernels 3/4

def test_isvd_stream_golden(golden):
    P = _pkg()
    g = golden("isvd")
    n, r, k, lam, steps = g["meta"]
    r = int(r)
    basis = P.ReducedBasis(phi=g["phi0"], sigma=g["sigma0"])
    for j, y in enumerate(g["stream"][r:]):
        basis = P.isvd_update(basis, y, float(lam), r)
        assert np.allclose(basis.sigma, g["sigma_hist"][j], rtol=1e-10, atol=0), j
    assert subspace.principal_angles(basis.phi, g["phiN"]).max() < 1e-10
    assert subspace.orthonormality_defect(basis.phi) < 1e-12


def test_isvd_known_answers(golden):
    P = _pkg()
    g = golden("isvd")
    out = P.isvd_update(P.ReducedBasis(np.eye(4)[:, :1], np.array([1.0])), np.eye(4)[:, 0], 1.0, 1)
    assert np.allclose(out.sigma, [np.sqrt(2.0)])
    assert np.allclose(np.abs(out.phi[:, 0]), np.eye(4)[:, 0])
    out = P.isvd_update(P.ReducedBasis(np.eye(5)[:, :2], np.array([2.0, 1.0])), np.zeros(5), 0.5, 2)
    assert np.allclose(out.sigma, [1.0, 0.5])
    assert subspace.orthonormality_defect(out.phi) <= 1e-12
    phi0 = g["ka_deg_phi0"]
    out = P.isvd_update(P.ReducedBasis(phi0, np.array([2.0, 1.0, 0.5])), g["ka_deg_y"], 0.9, 3)
    assert subspace.principal_angles(out.phi, phi0).max() <= 1e-12
    assert np.allclose(out.sigma, g["ka_deg_sigma"], rtol=1e-12)
    assert subspace.orthonormality_defect(out.phi) <= 1e-12
    # lambda = 0: sigma_1 = ||y|| (test_tracking.py:42-48)
    rng = np.random.default_rng(0)
    phi, _ = np.linalg.qr(rng.standard_normal((6, 2)))
    y = rng.standard_normal(6)
    out = P.isvd_update(P.ReducedBasis(phi, np.array([3.0, 1.0])), y, 0.0, 2)
    assert np.isclose(out.sigma[0], np.linalg.norm(y))


@pytest.mark.parametrize("n,r,lam", [(1 << 14, 16, 0.1), (1 << 16, 32, 0.25), (1 << 20, 64, 1.0)])
def test_isvd_vs_oracle(n, r, lam):
    P = _pkg()
    rng = np.random.default_rng(n + r)
    k = r + 32
    modes = np.linalg.qr(rng.standard_normal((n, k)))[0]
    spec = np.arange(1, k + 1) ** -1.5
    ys = [modes @ (spec * rng.standard_normal(k)) + 1e-6 * rng.standard_normal(n)
          for _ in range(r + 4)]
    u, s, _ = subspace.thin_svd(np.column_stack(ys[:r]))
    phi_c, sig_c = u[:, :r], s[:r]
    basis = P.ReducedBasis(phi=phi_c.copy(), sigma=sig_c.copy())
    for y in ys[r:]:
        phi_c, sig_c, _ = subspace.isvd_update(phi_c, sig_c, y, lam, r)
        basis = P.isvd_update(basis, y, lam, r)
        assert np.allclose(basis.sigma, sig_c, rtol=1e-9)
    assert subspace.max_angle(phi_c, basis.phi) < 1e-8


def test_isvd_device_tensors_stay_on_device():
    import torch
    P = _pkg()
    n, r = 1 << 18, 64
    g = torch.Generator(device="cuda").manual_seed(0)
    phi = torch.linalg.qr(torch.randn(n, r, dtype=torch.float64, device="cuda", generator=g))[0]
    sig = torch.linspace(10, 1, r, dtype=torch.float64, device="cuda")
    y = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    out = P.isvd_update(P.ReducedBasis(phi, sig), y, 0.5, r)
    assert out.phi.is_cuda and out.sigma.is_cuda
    ref_phi, ref_sig, _ = subspace.isvd_update(phi.cpu().numpy(), sig.cpu().numpy(),
                                               y.cpu().numpy(), 0.5, r, projection="gram")
    assert np.allclose(out.sigma.cpu().numpy(), ref_sig, rtol=1e-10)
    assert subspace.max_angle(ref_phi, out.phi.cpu().numpy()) < 1e-9


def test_isvd_rejects_nonfinite():
    P = _pkg()
    phi = np.eye(6)[:, :2]
    y = np.ones(6)
    y[3] = np.nan
    with pytest.raises(P.DenseError):
        P.isvd_update(P.ReducedBasis(phi, np.ones(2)), y, 0.5, 2)


@pytest.mark.parametrize("m,n", [(17, 17), (65, 65), (40, 7), (7, 40), (615, 32)])
def test_thin_svd_vs_numpy(m, n):
    P = _pkg()
    rng = np.random.default_rng(m * n)
    a = rng.standard_normal((m, n)) * np.logspace(0, -6, n)[None, :]
    res = P.thin_svd(a)
    s_ref = np.linalg.svd(a, compute_uv=False)
    assert np.allclose(res.s, s_ref, rtol=1e-12, atol=1e-14 * s_ref[0])
    assert np.allclose((res.u * res.s) @ res.v.T, a, atol=1e-12 * s_ref[0])


def test_encode_decode_vs_numpy():
    import ctypes as C
    import torch
    P = _pkg()
    from paper_2605_28684_b200 import _lib
    n, r = 100003, 16
    rng = np.random.default_rng(3)
    phi = np.linalg.qr(rng.standard_normal((n, r)))[0]
    q_ref = rng.standard_normal(n)
    d = np.tile(1.0 / np.array([2.0]), n)
    q = rng.standard_normal(n)
    ctx = _lib.Context.get()
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    a = torch.empty(r, dtype=torch.float64, device="cuda")
    tp, tq, td, tqq = t(phi), t(q_ref), t(d), t(q)
    ctx.call("adrom_encode", _lib.ptr(tp), _lib.ptr(tq), _lib.ptr(td), _lib.ptr(tqq),
             C.c_int64(n), C.c_int32(r), _lib.ptr(a))
    a_ref = phi.T @ (d * (q - q_ref))
    assert np.allclose(a.cpu().numpy(), a_ref, rtol=1e-12, atol=1e-12)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    ctx.call("adrom_decode", _lib.ptr(tp), _lib.ptr(tq), _lib.ptr(td), _lib.ptr(a), C.c_int64(n),
             C.c_int32(r), _lib.ptr(out))
    q_ref2 = q_ref + (phi @ a_ref) / d
    assert np.allclose(out.cpu().numpy(), q_ref2, rtol=1e-13, atol=1e-13)
