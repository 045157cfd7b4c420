"""Error path on the device (reference driver.py:168-199,
393-405): adrom_state_errors against numpy, and the replayed error pass of
run_adaptive_rom (per-step errors + signal errors) against the reference
loop's numbers and against a device ground truth that is never stored."""

import numpy as np
import pytest

from oracle import online, physics, subspace

pytestmark = pytest.mark.gpu


def _np_errors(model, pred, truth):
    from paper_2605_28684_b200.driver import _per_variable_errors
    return _per_variable_errors(model, pred, truth)


@pytest.mark.parametrize("kind", ["burgers", "sod", "reacting"])
def test_state_errors_match_numpy(kind):
    import torch
    import paper_2605_28684_b200 as P
    from paper_2605_28684_b200.driver import state_errors
    rng = np.random.default_rng(3)
    if kind == "burgers":
        m = P.BurgersProblem(5000, nu=1e-3)
    elif kind == "sod":
        m = P.SodProblem(3000)
    else:
        m = P.ReactingEulerProblem(2000)
    q = m.initial_state()
    pred = q * (1.0 + 1e-3 * rng.standard_normal(q.size))
    got = state_errors(m, torch.from_numpy(pred).cuda(), torch.from_numpy(q).cuda()).cpu().numpy()
    ref = _np_errors(m, pred, q)
    assert np.allclose(got, ref, rtol=1e-12, atol=0.0), (got, ref)
    zero = state_errors(m, torch.from_numpy(q).cuda(), torch.from_numpy(q).cuda()).cpu().numpy()
    assert np.all(zero == 0.0)


def test_error_pass_matches_reference_loop(golden):
    """loop_sod64_fgs: errors from the replayed session equal the reference's
    error history; signal errors equal those of the oracle loop's coarse
    snapshots (driver.py:398-405)."""
    import paper_2605_28684_b200 as P
    import test_gpu_rom as T
    name = "loop_sod64_fgs"
    g = golden(name)
    cfg = T._exp_config(name)
    res = P.run_adaptive_rom(cfg, truth=g["truth"], offline=T._oracle_offline(name, g))
    assert np.allclose(res.errors, g["errors"], rtol=1e-6, atol=1e-14)
    ocfg = online.LoopConfig(**T.LOOPS[name])
    training = g["truth"][: ocfg.w_init + 1]
    q_ref, d, phi0, sigma0 = online.offline(ocfg, training)
    rec = online.run_online(ocfg, training, q_ref, d, phi0, sigma0)
    model = P.make_problem(cfg)
    ref = [(s, _np_errors(model, y, g["truth"][s])) for s, y in rec.signal if s <= cfg.n_t]
    assert list(res.signal_steps) == [s for s, _ in ref]
    assert np.allclose(res.signal_errors, np.array([e for _, e in ref]), rtol=1e-8, atol=1e-14)
    assert res.time_averaged_signal_error("rho") == pytest.approx(
        float(np.mean([e[0] for _, e in ref])), rel=1e-8)


def test_device_truth_z1_signal_is_the_fine_truth():
    """Configuration-3 recipe (z = 1) at N = 2^18 without storing anything:
    truth="device" advances the fine FOM in lockstep; coarse_step(z = 1) is
    bitwise implicit_step(dt) (test_fom.py:211-216), so every signal error is
    exactly 0 and the per-step errors are those against the stored truth."""
    import paper_2605_28684_b200 as P
    import bench
    from paper_2605_28684_b200 import configs
    case = configs.cfg3(1 << 18, n_online=24)
    cfg, model = bench.rom_experiment(case)
    res = P.run_adaptive_rom(cfg, truth="device", problem=model, keep_every=0)
    assert res.errors.shape == (24, 1) and np.all(np.isfinite(res.errors))
    assert list(res.signal_steps) == list(range(case.w_init + 1, case.n_t + 1))
    assert np.all(res.signal_errors == 0.0)
    fom = P.run_fom(cfg, problem=model)
    res2 = P.run_adaptive_rom(cfg, truth=fom.trajectory, problem=model, keep_every=0)
    assert np.array_equal(res.errors, res2.errors)
