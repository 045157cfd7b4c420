"""Shared driver of the configuration-3 parity checks (the benchmarked recipe:
Burgers with the seeded bump IC, CFL-0.4 dt, r = n_s = 64, z = 1, lambda = 0.1,
LSPG + QDEIM, an iSVD event after every online step).

The oracle (``oracle.online.run_online``, the restatement of the reference's
``driver._run_rom``) and the device session run the same online loop from
identical offline inputs (the oracle's training window, scaling and POD,
which the reference computes outside its timed region).  Everything the loop
decides or produces is compared step by step: decoded states, Gauss-Newton
iteration counts, coarse Newton iteration counts, QDEIM rows, singular
values.

Also runnable as a diagnostic on the GPU box:

    python tests/cfg3_parity.py --n 65536 --steps 200
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from oracle import online, physics, subspace  # noqa: E402


def oracle_setup(n: int, steps: int):
    from paper_2605_28684_b200 import configs
    case = configs.cfg3(n, n_online=steps)
    m = physics.Model("burgers", n, nu=case.nu)
    ocfg = online.LoopConfig(model=m, dt=case.dt, n_t=case.n_t, w_init=case.w_init, r=case.r,
                             n_s=case.n_s, z=case.z, lam=case.lam)
    training = online.training_states(ocfg, case.initial_state())
    q_ref, phi_norm = subspace.fit_scaling(list(training), 1)
    _, d, phi0, sigma0 = online.offline(ocfg, training)
    return case, ocfg, training, q_ref, phi_norm, d, phi0, sigma0


def oracle_run(setup, steps, nudge_seed=None, pinned=None, nudge_ulps=1.0):
    case, ocfg, training, q_ref, phi_norm, d, phi0, sigma0 = setup
    return online.run_online(ocfg, training, q_ref, d, phi0, sigma0, keep_stride=1,
                             n_steps=steps, nudge_seed=nudge_seed, pinned_samplings=pinned,
                             nudge_ulps=nudge_ulps)


def envelope(setup, steps, ref, seeds=(1, 2, 3)):
    """Per-step relative state spread and per-event sigma spread of the
    oracle loop under one-ulp nudges (max over seeds)."""
    states = np.array(ref.states)
    sig = np.array(ref.sigma)
    env_s = np.zeros(len(states))
    env_sig = np.zeros(sig.shape)
    for s in seeds:
        rec = oracle_run(setup, steps, nudge_seed=s)
        st = np.array(rec.states)
        env_s = np.maximum(env_s, np.linalg.norm(st - states, axis=1) / np.linalg.norm(states, axis=1))
        env_sig = np.maximum(env_sig, np.abs(np.array(rec.sigma) - sig) / np.abs(sig))
    return env_s, env_sig


def gpu_run(setup, steps, stepwise=True, keep_phi_at=()):
    """The device session from the oracle's offline results; returns the
    decoded state, iteration count, sampled rows and sigma of every step."""
    import torch
    import paper_2605_28684_b200 as P
    import bench
    from paper_2605_28684_b200.driver import Session
    case, ocfg, training, q_ref, phi_norm, d, phi0, sigma0 = setup
    cfg, model = bench.rom_experiment(case)
    sess = Session(cfg, model, adaptive=True)
    scaling = P.ScalingTransform(q_ref=q_ref, phi_norm=phi_norm)
    sess.load(scaling, P.ReducedBasis(phi=phi0, sigma=sigma0), training[case.w_init])
    sess.start()
    out = torch.empty((steps, model.n_dof), dtype=torch.float64, device="cuda")
    samp = [sess.sampling().cpu().numpy().copy()]
    sig = []
    phis = {}
    if stepwise:
        for k in range(steps):
            sess.advance(1, 1, out[k:k + 1], None)
            _, _, _, s, _ = sess.read(1, 1)
            sig.append(s.cpu().numpy().copy())
            samp.append(sess.sampling().cpu().numpy().copy())
            if k + 1 in keep_phi_at:
                phis[k + 1] = sess.basis().cpu().numpy()
    else:
        sess.advance(steps, 1, out, None)
    sess.finish()
    log, ev, a, s_fin, _ = sess.read(steps, steps)
    phi = sess.basis().cpu().numpy()
    sess.close()
    return dict(traj=out.cpu().numpy(), it=log[:, 1].astype(int).copy(),
                conv=log[:, 0].copy(),
                coarse=[int(e.coarse_iterations) for e in ev],
                errors=[int(e.error) for e in ev], sig=np.array(sig), samp=samp, phi=phi,
                phis=phis)


def restart_parity(setup, steps_at, n_steps=2):
    """Local (per-step) parity along the trajectory: at each checkpoint the
    oracle's state after the event of online step ``st`` (1-based; basis,
    sigma, decoded state) restarts BOTH
    loops (start: coarse lookahead, QDEIM, operator, encode; then n_steps
    online steps).  The configuration-3 loop is chaotic under rounding (an
    ulp nudge grows to O(1) within ~100 steps, tests/golden/cfg3_envelope.npz)
    so a long trajectory cannot be compared pointwise; every step map can."""
    import paper_2605_28684_b200 as P
    case, ocfg, training, q_ref, phi_norm, d, phi0, sigma0 = setup
    last = max(steps_at)
    full = online.run_online(ocfg, training, q_ref, d, phi0, sigma0, keep_stride=10 ** 9,
                             n_steps=last, checkpoint_steps={case.w_init + s for s in steps_at})
    out = []
    for st in steps_at:
        phi_s, sig_s, q_s = full.checkpoints[case.w_init + st]
        rec = online.run_online(ocfg, {case.w_init: q_s}, q_ref, d, phi_s, sig_s, keep_stride=1,
                                n_steps=n_steps)
        sub = (case, ocfg, {case.w_init: q_s}, q_ref, phi_norm, d, phi_s, sig_s)
        got = gpu_run(sub, n_steps)
        rep = compare(rec, got)
        rep["step"] = st
        out.append(rep)
    return out


def trajectory_step_parity(setup, steps, every=1):
    """Step-map parity along the DEVICE loop's own trajectory: after every
    ``every``-th online step, both implementations restart from the device
    state (basis and singular values after the step's event, decoded state)
    and run one step + its event.  The loop is chaotic under rounding (an
    ulp nudge grows to O(1e-2) over 200 steps, and the Gauss-Newton solve
    of some states oscillates for all 10 iterations in both implementations),
    so a long free-running trajectory cannot be compared pointwise; this
    compares every step map the device trajectory actually visits."""
    import torch
    case, ocfg, training, q_ref, phi_norm, d, phi0, sigma0 = setup
    got = gpu_run(setup, steps, keep_phi_at=set(range(every, steps + 1, every)))
    out = []
    for k in sorted(got["phis"]):
        phi_k = got["phis"][k]
        sig_k = got["sig"][k - 1]
        q_k = got["traj"][k - 1]
        sub = (case, ocfg, {case.w_init: q_k}, q_ref, phi_norm, d, phi_k, sig_k)
        rec = online.run_online(ocfg, {case.w_init: q_k}, q_ref, d, phi_k, sig_k, keep_stride=1,
                                n_steps=1)
        g = gpu_run(sub, 1)
        rep = compare(rec, g)
        rep["step"] = k
        out.append(rep)
        del g
    torch.cuda.empty_cache()
    return out, got


def compare(ref, got, env_s=None, env_sig=None):
    """Deviation report (dict of arrays) of the device loop vs the oracle."""
    states = np.array(ref.states)
    dev = np.linalg.norm(got["traj"] - states, axis=1) / np.linalg.norm(states, axis=1)
    it_ref = np.array(ref.iterations)
    rep = dict(dev=dev, it_ref=it_ref, it_got=got["it"],
               coarse_ref=[e["coarse_iterations"] for e in ref.events],
               coarse_conv_ref=[bool(e.get("coarse_converged", True)) for e in ref.events],
               coarse_got=got["coarse"], event_errors=got["errors"],
               fail_ref=list(ref.failures))
    if len(got["sig"]):
        sig_ref = np.array(ref.sigma)
        rep["sig_rel"] = np.abs(got["sig"] - sig_ref) / sig_ref
        rep["sig_abs1"] = np.abs(got["sig"] - sig_ref) / sig_ref[:, :1]
        rep["samp_equal"] = np.array([np.array_equal(np.sort(a), np.sort(b))
                                      for a, b in zip(ref.samplings, got["samp"])])
    rep["angle_final"] = subspace.max_angle(ref.phi_final, got["phi"])
    return rep


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 16)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--envelope", type=int, default=0, help="number of nudge seeds")
    a = ap.parse_args(argv)
    t0 = time.time()
    setup = oracle_setup(a.n, a.steps)
    print(f"oracle offline {time.time() - t0:.1f}s sigma0[:4]={setup[-1][:4]}", flush=True)
    t0 = time.time()
    ref = oracle_run(setup, a.steps)
    print(f"oracle online {time.time() - t0:.1f}s", flush=True)
    t0 = time.time()
    got = gpu_run(setup, a.steps)
    print(f"gpu {time.time() - t0:.1f}s", flush=True)
    rep = compare(ref, got)
    print("state dev max", rep["dev"].max(), "at", int(rep["dev"].argmax()))
    print("state dev per 10 steps", rep["dev"][::10])
    print("GN its ref", rep["it_ref"][:20], "mean", rep["it_ref"].mean())
    print("GN its gpu", rep["it_got"][:20], "mean", rep["it_got"].mean())
    print("coarse its equal", rep["coarse_ref"] == rep["coarse_got"], "event errors", sum(rep["event_errors"]))
    print("failures ref", rep["fail_ref"][:10], len(rep["fail_ref"]))
    print("sigma rel max (sig>1e-8 s1)", np.max(np.where(np.array(ref.sigma) > 1e-8 * np.array(ref.sigma)[:, :1], rep["sig_rel"], 0)))
    print("sigma abs/s1 max", rep["sig_abs1"].max())
    print("sampling equal", rep["samp_equal"].sum(), "/", len(rep["samp_equal"]))
    print("final angle", rep["angle_final"])
    if a.envelope:
        env_s, env_sig = envelope(setup, a.steps, ref, seeds=tuple(range(1, a.envelope + 1)))
        print("envelope state max", env_s.max(), "per 10", env_s[::10])


if __name__ == "__main__":
    main()
