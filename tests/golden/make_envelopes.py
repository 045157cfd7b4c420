"""Rounding-sensitivity envelopes of the configuration-1 and -3 loops, from
the oracle's restatement of the reference loop (the reference's own driver
cannot run at these sizes: dense N^2 Newton).

Protocol (``oracle.online.run_online(nudge_seed=..., nudge_ulps=u)``), three
seeds each for u = 1 and u = 8: every coarse Newton result, iSVD basis,
reduced step and state transfer is perturbed by one ulp (u = 1) or by up to
8 ulps relative with every singular value moved by up to 8 eps sigma_1
absolute (u = 8: the accuracy LAPACK's gesdd guarantees for the core SVD —
backward stability; 8 eps ||K|| is also its deflation tolerance — which a
one-ulp relative nudge understates: the reference reproduces its own tiny
singular values far more tightly than it computes them).  The envelope is
the max over all runs of the per-step relative state spread and the
per-event singular-value spread; decisions (sampled rows, iteration counts)
count as stable where no run changed them.

    python tests/golden/make_envelopes.py [cfg1] [cfg3]
"""

import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(OUT.parents[1]))
sys.path.insert(0, str(OUT.parent))

from oracle import online, physics, subspace  # noqa: E402

ULPS = (1.0, 8.0)   # one-ulp nudges and the LAPACK-accuracy perturbation
SEEDS = (1, 2, 3)


def _envelope(name, ocfg, training, q_ref, d, phi0, sigma0, steps, extra):
    ref = online.run_online(ocfg, training, q_ref, d, phi0, sigma0, keep_stride=1, n_steps=steps)
    states = np.array(ref.states)
    sig = np.array(ref.sigma)
    env_s = np.zeros(len(states))
    env_sig = np.zeros(sig.shape)
    stable = np.ones(len(ref.samplings), dtype=bool)
    its_stable = np.ones(len(ref.iterations), dtype=bool)
    for ulps, s in [(u, s) for u in ULPS for s in SEEDS]:
        rec = online.run_online(ocfg, training, q_ref, d, phi0, sigma0, keep_stride=1,
                                n_steps=steps, nudge_seed=s, nudge_ulps=ulps)
        st = np.array(rec.states)
        env_s = np.maximum(env_s, np.linalg.norm(st - states, axis=1) / np.linalg.norm(states, axis=1))
        env_sig = np.maximum(env_sig, np.abs(np.array(rec.sigma) - sig) / np.abs(sig))
        for k, (x, y) in enumerate(zip(rec.samplings, ref.samplings)):
            if not np.array_equal(np.sort(x), np.sort(y)):
                stable[k] = False
        its_stable &= np.array(rec.iterations) == np.array(ref.iterations)
        print(f"{name} ulps {ulps} seed {s}: state spread max {env_s.max():.3e}", flush=True)
    np.savez_compressed(OUT / f"{name}_envelope.npz", steps=np.array(steps), ulps=np.array(ULPS),
                        env_state=env_s, env_sigma=env_sig, samp_stable=stable,
                        its_stable=its_stable, iterations=np.array(ref.iterations), **extra)
    print(f"wrote {name}_envelope.npz; stable events {stable.mean():.2f}")


def cfg1(steps=200):
    from paper_2605_28684_b200 import configs
    case = configs.cfg1()
    m = physics.Model("sod", case.n_elem, gamma=case.gamma)
    ocfg = online.LoopConfig(model=m, dt=case.dt, n_t=case.w_init + steps, w_init=case.w_init,
                             r=case.r, n_s=case.n_s, z=case.z, lam=case.lam,
                             projection=case.projection, sampling=case.sampling,
                             feature=case.feature, n_extra=case.n_extra)
    training = online.training_states(ocfg, case.initial_state())
    _, d, phi0, sigma0 = online.offline(ocfg, training)
    q_ref, _ = subspace.fit_scaling(list(training), m.n_var)
    _envelope("cfg1", ocfg, training, q_ref, d, phi0, sigma0, steps, {"n": np.array(case.n_elem)})


def cfg3(n=1 << 16, steps=200):
    import cfg3_parity as C
    case, ocfg, training, q_ref, phi_norm, d, phi0, sigma0 = C.oracle_setup(n, steps)
    _envelope("cfg3", ocfg, training, q_ref, d, phi0, sigma0, steps, {"n": np.array(n)})


if __name__ == "__main__":
    for w in sys.argv[1:] or ["cfg1", "cfg3"]:
        globals()[w]()
