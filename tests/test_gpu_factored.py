"""The session's factored basis (csrc/factored.cu): Phi = [A | Q] W instead of
an explicit rotation every event.  It is the default for r in {32, 64} at
N >= 2^18; ADROM_FACTORED=1/0 forces it on/off.  These tests run the same
loop both ways and against the oracle (the reference's algorithm)."""

import os

import numpy as np
import pytest

import bench
from oracle import online, physics, subspace

pytestmark = pytest.mark.gpu


def _run(case, steps, fact, offline=None):
    import torch
    import paper_2605_28684_b200 as P
    from paper_2605_28684_b200.driver import Session, offline_stage
    old = os.environ.get("ADROM_FACTORED")
    os.environ["ADROM_FACTORED"] = "1" if fact else "0"
    try:
        cfg, model = bench.rom_experiment(case)
        training, scaling, basis0 = offline_stage(cfg, model)
        if offline is not None:
            scaling, basis0 = offline
        sess = Session(cfg, model, adaptive=True)
        sess.load(scaling, basis0, training[cfg.w_init])
        sess.start()
        out = torch.empty((steps, model.n_dof), dtype=torch.float64, device="cuda")
        sess.advance(steps, 1, out, None)
        sess.finish()
        log, ev, a, sig, q = sess.read(steps, steps)
        idx = np.sort(sess.sampling().cpu().numpy())
        phi = sess.basis().cpu().numpy()
        sess.close()
    finally:
        if old is None:
            os.environ.pop("ADROM_FACTORED", None)
        else:
            os.environ["ADROM_FACTORED"] = old
    return dict(traj=out.cpu().numpy(), it=log[:, 1].copy(),
                ev=[(int(e.step), int(e.error), int(e.coarse_iterations)) for e in ev],
                sig=sig.cpu().numpy(), idx=idx, phi=phi)


@pytest.mark.parametrize("name,n,steps,tol", [
    ("cfg1", 4096, 40, 1e-10),     # Sod, r = 32, FGS: well conditioned
    ("cfg3", 1 << 16, 40, 1e-6),   # Burgers, r = 64, z = 1: ~59 noise directions,
                                   # 40 events = 2 re-anchors
    ("cfg3", 1 << 18, 20, 1e-6),   # above the all-rows pool limit: the factored
])                                 # refresh of the certified QDEIM pool
def test_factored_matches_explicit(name, n, steps, tol):
    case = bench.rom_case(name, n)
    e = _run(case, steps, fact=False)
    f = _run(case, steps, fact=True)
    dev = np.linalg.norm(e["traj"] - f["traj"], axis=1) / np.linalg.norm(e["traj"], axis=1)
    assert dev.max() <= tol, dev.max()
    assert np.array_equal(e["it"], f["it"])
    assert e["ev"] == f["ev"] and all(err == 0 for _, err, _ in f["ev"])
    assert np.array_equal(e["idx"], f["idx"])
    big = e["sig"] > 1e-8 * e["sig"][0]
    assert np.max(np.abs(e["sig"] - f["sig"])[big] / e["sig"][big]) <= 1e-8
    # the materialised basis is as orthonormal as the explicitly rotated one
    # (noise-level K directions make both drift; the Gram matrix is tracked)
    de, df = subspace.orthonormality_defect(e["phi"]), subspace.orthonormality_defect(f["phi"])
    assert df <= 10.0 * de + 1e-11, (de, df)


def test_factored_vs_oracle_sod():
    """cfg1 (Sod, r = 32, FGS) on the factored basis against the oracle's
    restatement of driver._run_rom, both from the oracle's POD."""
    import paper_2605_28684_b200 as P
    case = bench.rom_case("cfg1", 4096)
    steps = 20
    m = physics.Model("sod", case.n_elem, gamma=case.gamma)
    ocfg = online.LoopConfig(model=m, dt=case.dt, n_t=case.w_init + steps + 1, w_init=case.w_init,
                             r=case.r, n_s=case.n_s, z=case.z, lam=case.lam,
                             projection=case.projection, sampling=case.sampling,
                             feature=case.feature, n_extra=case.n_extra)
    training = online.training_states(ocfg, case.initial_state())
    q_ref, phi_norm = subspace.fit_scaling(list(training), m.n_var)
    _, d, phi0, sigma0 = online.offline(ocfg, training)
    rec = online.run_online(ocfg, training, q_ref, d, phi0, sigma0, keep_stride=1, n_steps=steps)
    off = (P.ScalingTransform(q_ref=q_ref, phi_norm=phi_norm), P.ReducedBasis(phi=phi0, sigma=sigma0))
    f = _run(case, steps, fact=True, offline=off)
    ref = np.array(rec.states)
    dev = np.linalg.norm(f["traj"] - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert dev.max() <= 1e-8, dev.max()
    assert np.array_equal(np.sort(rec.samplings[-1]), f["idx"])
    assert subspace.max_angle(rec.phi_final, f["phi"]) < 1e-8


@pytest.mark.parametrize("n,r,lam", [(1 << 16, 64, 1.0), (1 << 15, 32, 0.5)])
def test_isvd_stream_matches_repeated_updates(n, r, lam):
    """IsvdStream (factored, 40 updates = 2 re-anchors) against the explicit
    isvd_update chain and against the oracle's restatement of tracking.py."""
    import paper_2605_28684_b200 as P
    rng = np.random.default_rng(n + r)
    k = r + 32
    modes = np.linalg.qr(rng.standard_normal((n, k)))[0]
    spec = np.arange(1, k + 1) ** -1.5
    ys = [modes @ (spec * rng.standard_normal(k)) + 1e-6 * rng.standard_normal(n)
          for _ in range(r + 40)]
    u, s, _ = subspace.thin_svd(np.column_stack(ys[:r]))
    b0 = P.ReducedBasis(phi=u[:, :r].copy(), sigma=s[:r].copy())
    stream = P.tracking.IsvdStream(b0)
    basis = b0
    phi_c, sig_c = u[:, :r].copy(), s[:r].copy()
    for y in ys[r:]:
        stream.update(y, lam)
        basis = P.isvd_update(basis, y, lam, r)
        phi_c, sig_c, _ = subspace.isvd_update(phi_c, sig_c, y, lam, r)
    got = stream.basis()
    sig_f = got.sigma.cpu().numpy()
    phi_f = got.phi.cpu().numpy()
    assert np.allclose(sig_f, np.asarray(basis.sigma), rtol=1e-10)
    assert np.allclose(sig_f, sig_c, rtol=1e-9)
    assert subspace.max_angle(phi_c, phi_f) < 1e-8
    assert subspace.max_angle(np.asarray(basis.phi), phi_f) < 1e-9
    assert subspace.orthonormality_defect(phi_f) <= 1e-11
    stream.close()


def test_isvd_stream_rejects_nonfinite():
    import paper_2605_28684_b200 as P
    from paper_2605_28684_b200.errors import DenseError
    n, r = 4096, 32
    rng = np.random.default_rng(1)
    phi = np.linalg.qr(rng.standard_normal((n, r)))[0]
    st = P.tracking.IsvdStream(P.ReducedBasis(phi=phi, sigma=np.linspace(2, 1, r)))
    st.update(rng.standard_normal(n), 0.9)
    before = st.basis()
    bad = rng.standard_normal(n)
    bad[7] = np.nan
    with pytest.raises(DenseError):
        st.update(bad, 0.9)
    after = st.basis()
    assert np.array_equal(before.sigma.cpu().numpy(), after.sigma.cpu().numpy())
    assert np.array_equal(before.phi.cpu().numpy(), after.phi.cpu().numpy())
    st.close()
