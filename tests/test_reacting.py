"""Configuration-4 reacting Euler residual.

The reference has no reacting model, so parity is UNPINNED: the
oracle (oracle/reacting.py) defines the model, and the CUDA kernel is checked
against it plus the conservation identities the model guarantees.
"""

import numpy as np
import pytest

from oracle import reacting as R


def _pkg():
    import paper_2605_28684_b200 as P
    return P


def test_mechanism_and_ic_match_oracle():
    P = _pkg()
    m = P.ReactingEulerProblem(257)
    assert np.array_equal(m.mechanism, R.mechanism(4))
    assert np.array_equal(m.initial_state(), R.initial_state(257))
    mech = m.mechanism
    assert np.all(mech[0] != mech[1])  # no self-reactions
    assert m.n_var == 13 and m.n_dof == 257 * 13


@pytest.mark.parametrize("n", [4, 7, 1024])
def test_oracle_conservation(n):
    q = R.initial_state(n)
    f = R.rhs(q, n, 1.0 / n, 1.4, R.mechanism()).reshape(n, R.N_VAR)
    scale = np.abs(f).max()
    # periodic flux differences telescope; reactions only move species mass
    assert abs(f[:, 0].sum()) <= 1e-12 * scale * n
    assert abs(f[:, 1].sum()) <= 1e-12 * scale * n
    assert abs(f[:, 3:].sum()) <= 1e-12 * scale * n
    # energy changes only by the heat release
    src = R.sources(q.reshape(n, R.N_VAR), 1.4, R.mechanism())
    assert abs(f[:, 2].sum() - src[:, 2].sum()) <= 1e-12 * scale * n


def test_oracle_uniform_state_without_reactions_is_equilibrium():
    mech = R.mechanism().copy()
    mech[2] = 0.0
    cell = R.initial_state(4).reshape(4, R.N_VAR)[0]
    q = np.tile(cell, 16)
    assert np.all(R.rhs(q, 16, 1.0 / 16, 1.4, mech) == 0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [4, 5, 129, 1000, 1 << 16])
def test_reacting_rhs_vs_oracle(n):
    P = _pkg()
    m = P.ReactingEulerProblem(n)
    q = m.initial_state()
    rng = np.random.default_rng(n)
    q = q * (1.0 + 0.01 * rng.standard_normal(q.size))
    got = np.asarray(m.rhs(q))
    ref = R.rhs(q, n, m.dx, m.gamma, m.mechanism)
    # same operation order as the oracle (--fmad=false); exp() may differ by
    # an ulp between CUDA and numpy, so the gate is normwise 1e-13
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= 1e-13, err
    # the flux part is exact: compare with the reactions switched off
    f = got.reshape(n, 13)
    scale = np.abs(f).max()
    assert abs(f[:, 0].sum()) <= 1e-11 * scale * n
    assert abs(f[:, 3:].sum()) <= 1e-11 * scale * n


@pytest.mark.gpu
def test_reacting_rhs_device_resident_and_errors():
    P = _pkg()
    import torch
    m = P.ReactingEulerProblem(4096)
    q = torch.from_numpy(m.initial_state()).cuda()
    f = m.rhs(q)
    assert f.is_cuda and f.shape == q.shape
    ref = R.rhs(m.initial_state(), 4096, m.dx, m.gamma, m.mechanism)
    assert np.linalg.norm(f.cpu().numpy() - ref) <= 1e-13 * np.linalg.norm(ref)
    with pytest.raises(ValueError):
        m.rhs(np.zeros(5))


@pytest.mark.gpu
@pytest.mark.parametrize("n", [7, 64])
def test_reacting_fd_jacobian_vs_oracle(n):
    """Banded FD Jacobian (the reference's colouring scheme, fom.py:301-328,
    on the builder-defined model).  The difference quotients amplify the
    ulp-level exp() differences by 1/eps: normwise 1e-7 per block row."""
    P = _pkg()
    from oracle import physics
    m = P.ReactingEulerProblem(n)
    q = m.initial_state() * (1.0 + 0.01 * np.random.default_rng(n).standard_normal(n * 13))
    om = physics.Model("reacting", n, gamma=1.4, mech=tuple(m.mechanism.ravel()))
    ref = physics.fd_jacobian_blocks(om, q)
    got = np.asarray(P.fd_jacobian_blocks(m, q))
    assert got.shape == ref.shape
    err = np.linalg.norm((got - ref).reshape(n, -1), axis=1) / np.linalg.norm(ref.reshape(n, -1), axis=1)
    assert err.max() <= 1e-7, err.max()


@pytest.mark.gpu
@pytest.mark.parametrize("n,dt", [(64, 1e-3), (1000, 2e-4)])
def test_reacting_implicit_step_vs_oracle(n, dt):
    """Backward-Euler Newton on the reacting model (a4 for configuration 4):
    13 x 13 block-tridiagonal cyclic solve on the device vs the oracle's
    sparse LU of the same matrix."""
    P = _pkg()
    from oracle import physics
    m = P.ReactingEulerProblem(n)
    q = m.initial_state()
    om = physics.Model("reacting", n, gamma=1.4, mech=tuple(m.mechanism.ravel()))
    ref = physics.implicit_step(om, q, dt)
    res = P.implicit_step(m, q, dt)
    assert res.converged == ref.converged and res.iterations == ref.iterations
    assert np.linalg.norm(np.asarray(res.x) - ref.x) <= 1e-12 * np.linalg.norm(ref.x)


def test_oracle_sampled_residual_equals_full_residual():
    """SamplingPlan.evaluate over every row == rhs, bitwise (the property the
    reference has for Burgers and Sod), for the reacting model."""
    from oracle import hyper, physics
    n = 40
    m = physics.Model("reacting", n, gamma=1.4, mech=tuple(R.mechanism().ravel()))
    q = R.initial_state(n) * (1.0 + 0.01 * np.sin(np.arange(n * R.N_VAR)))
    s = hyper.closure(hyper.Sampling(indices=np.arange(n * R.N_VAR), closure=None), m)
    plan = hyper.gather_plan(m, s)
    assert np.array_equal(plan.evaluate(m, q[s.closure]), physics.rhs(m, q))
