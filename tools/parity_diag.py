"""Diagnostics behind tests/test_gpu_parity_configs.py (prints instead of
asserting): cfg1 200-step loop with per-event decisions, cfg3 restarts."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def cfg1(steps=200, seeds=3):
    import bench
    import paper_2605_28684_b200 as P
    from oracle import online, physics, subspace
    import test_gpu_parity_configs as T
    case = bench.rom_case("cfg1", 4096)
    m = physics.Model("sod", case.n_elem, gamma=case.gamma)
    ocfg = online.LoopConfig(model=m, dt=case.dt, n_t=case.w_init + steps, w_init=case.w_init,
                             r=case.r, n_s=case.n_s, z=case.z, lam=case.lam,
                             projection=case.projection, sampling=case.sampling,
                             feature=case.feature, n_extra=case.n_extra)
    training = online.training_states(ocfg, case.initial_state())
    q_ref, phi_norm = subspace.fit_scaling(list(training), m.n_var)
    _, d, phi0, sigma0 = online.offline(ocfg, training)
    rec = online.run_online(ocfg, training, q_ref, d, phi0, sigma0, keep_stride=1, n_steps=steps)
    ref = np.array(rec.states)
    got = T._session(case, P.ScalingTransform(q_ref=q_ref, phi_norm=phi_norm),
                     P.ReducedBasis(phi=phi0, sigma=sigma0), training[case.w_init], steps, case.z)
    dev = np.linalg.norm(got["traj"] - ref, axis=1) / np.linalg.norm(ref, axis=1)
    print("cfg1 dev per 5 steps", np.array2string(dev[4::5], precision=2))
    eq = [np.array_equal(np.sort(a), np.sort(b)) for a, b in zip(got["samp"], rec.samplings)]
    print("cfg1 sampling equal per event", np.array(eq).astype(int))
    for k, (a, b) in enumerate(zip(got["samp"], rec.samplings)):
        if not eq[k]:
            print("  first differing event", k, "gpu-only", sorted(set(a) - set(b))[:10],
                  "ref-only", sorted(set(b) - set(a))[:10])
            break
    stab = np.ones(len(rec.samplings), bool)
    env = np.zeros(steps)
    for s in range(1, seeds + 1):
        e = online.run_online(ocfg, training, q_ref, d, phi0, sigma0, keep_stride=1, n_steps=steps,
                              nudge_seed=s)
        env = np.maximum(env, np.linalg.norm(np.array(e.states) - ref, axis=1) / np.linalg.norm(ref, axis=1))
        stab &= np.array([np.array_equal(np.sort(a), np.sort(b)) for a, b in zip(e.samplings, rec.samplings)])
    print("cfg1 envelope per 5 steps", np.array2string(env[4::5], precision=2))
    print("cfg1 ref sampling stable per event", stab.astype(int))
    print("its equal", np.mean(got["it"] == np.array(rec.iterations)))
    sr = np.array(rec.sigma)
    rel = np.abs(got["sig"] - sr) / sr
    print("cfg1 sigma rel dev (top 8 / all, per event)")
    for k in range(len(sr)):
        print(f"  ev {k:2d} top8 {rel[k, :8].max():.2e} all {rel[k].max():.2e} abs/s1 "
              f"{(np.abs(got['sig'][k] - sr[k]) / sr[k, 0]).max():.2e} coarse "
              f"{int(got['events'][k].coarse_iterations)}/{rec.events[k]['coarse_iterations']} "
              f"s_min/s1 {sr[k, -1] / sr[k, 0]:.1e}")


def cfg3():
    import cfg3_parity as C
    setup = C.oracle_setup(1 << 16, 200)
    reps = C.restart_parity(setup, list(range(1, 200, 20)), n_steps=2)
    for rep in reps:
        print("restart", rep["step"], "samp", rep["samp_equal"].astype(int), "dev",
              np.array2string(rep["dev"], precision=2), "its", rep["it_got"], rep["it_ref"],
              "coarse", rep["coarse_got"], rep["coarse_ref"], "sig_abs1", rep["sig_abs1"].max())


if __name__ == "__main__":
    for w in sys.argv[1:] or ["cfg1", "cfg3"]:
        globals()[w]()
