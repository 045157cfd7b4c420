"""Configuration 3 at its true size (N = 2^24): the first K online steps of the
device session against the oracle's restatement of the reference loop, both
from the same offline results (training window, scaling and POD computed
once on the device; the reference computes them before its timed region).

Also times every oracle component of those steps on the host cores — the
reference's own algorithms (gelsd iSVD, geqp3 QDEIM, the banded Newton
restatement, numpy residual/encode/decode) at the benchmarked size.

    python tools/cfg3_fulln_prefix.py --steps 3 --out gpurun_out/c3_fulln.json
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--n", type=int, default=1 << 24)
    ap.add_argument("--out", default="gpurun_out/c3_fulln.json")
    a = ap.parse_args(argv)
    import torch
    import bench
    import paper_2605_28684_b200 as P
    from paper_2605_28684_b200 import configs
    from paper_2605_28684_b200.driver import Session, offline_stage
    from oracle import hyper, online, physics, reduced, subspace

    case = configs.cfg3(a.n, n_online=a.steps)
    cfg, model = bench.rom_experiment(case)
    t0 = time.time()
    training, scaling, basis0 = offline_stage(cfg, model)
    q_last = training[cfg.w_init].clone()
    del training
    torch.cuda.synchronize()
    print(f"device offline {time.time() - t0:.1f}s", flush=True)

    # device session, one step at a time
    sess = Session(cfg, model, adaptive=True)
    sess.load(scaling, basis0, q_last)
    sess.start()
    samp_g = [sess.sampling().cpu().numpy().copy()]
    traj_g, sig_g = [], []
    out = torch.empty((1, model.n_dof), dtype=torch.float64, device="cuda")
    for _ in range(a.steps):
        sess.advance(1, 1, out, None)
        traj_g.append(out[0].cpu().numpy().copy())
        _, _, _, s, _ = sess.read(1, 1)
        sig_g.append(s.cpu().numpy().copy())
        samp_g.append(sess.sampling().cpu().numpy().copy())
    sess.finish()
    log, ev, _, _, _ = sess.read(a.steps, a.steps)
    sess.close()
    print("device GN iterations", log[:, 1], "converged", log[:, 0], flush=True)

    # host copies of the shared offline results
    q_ref = scaling.q_ref.cpu().numpy()
    phi_norm = scaling.phi_norm.cpu().numpy()
    d = np.tile(1.0 / phi_norm, case.n_elem)
    phi0 = basis0.phi.cpu().numpy()
    sigma0 = basis0.sigma.cpu().numpy()
    ql = q_last.cpu().numpy()
    del basis0, scaling, q_last
    torch.cuda.empty_cache()

    m = physics.Model("burgers", case.n_elem, nu=case.nu)
    ocfg = online.LoopConfig(model=m, dt=case.dt, n_t=case.n_t, w_init=case.w_init, r=case.r,
                             n_s=case.n_s, z=case.z, lam=case.lam)

    # component timings (the reference's algorithms at the benchmarked size)
    tm = {}

    def timed(name, fn, *args, **kw):
        t = time.perf_counter()
        out = fn(*args, **kw)
        tm.setdefault(name, []).append(time.perf_counter() - t)
        return out

    orig = (physics.coarse_step, subspace.isvd_update, hyper.qdeim, reduced.build_operator,
            reduced.encode, reduced.decode, reduced.lspg_step)
    online.physics.coarse_step = lambda *x, **k: timed("coarse_step", orig[0], *x, **k)
    online.subspace.isvd_update = lambda *x, **k: timed("isvd_update", orig[1], *x, **k)
    online.hyper.qdeim = lambda *x, **k: timed("qdeim_sample", orig[2], *x, **k)
    online.reduced.build_operator = lambda *x, **k: timed("build_operator", orig[3], *x, **k)
    online.reduced.encode = lambda *x, **k: timed("encode", orig[4], *x, **k)
    online.reduced.decode = lambda *x, **k: timed("decode", orig[5], *x, **k)
    online.reduced.lspg_step = lambda *x, **k: timed("lspg_step", orig[6], *x, **k)
    t0 = time.perf_counter()
    rec = online.run_online(ocfg, {case.w_init: ql}, q_ref, d, phi0, sigma0, keep_stride=1,
                            n_steps=a.steps)
    wall = time.perf_counter() - t0
    print(f"oracle online {wall:.1f}s", {k: [round(x, 3) for x in v] for k, v in tm.items()},
          flush=True)

    states = np.array(rec.states)
    dev = np.linalg.norm(np.array(traj_g) - states, axis=1) / np.linalg.norm(states, axis=1)
    sig_r = np.array(rec.sigma)
    rep = {
        "n_elem": case.n_elem, "steps": a.steps, "dt": case.dt,
        "state_rel_dev": dev.tolist(),
        "gn_iterations_oracle": [int(x) for x in rec.iterations],
        "gn_iterations_device": [int(x) for x in log[:, 1]],
        "failures_oracle": [int(x) for x in rec.failures],
        "converged_device": [int(x) for x in log[:, 0]],
        "coarse_iterations_oracle": [e.get("coarse_iterations") for e in rec.events],
        "coarse_iterations_device": [int(e.coarse_iterations) for e in ev],
        "sampling_equal": [bool(np.array_equal(np.sort(x), np.sort(y)))
                           for x, y in zip(rec.samplings, samp_g)],
        "sigma_rel_dev_max": [float(np.max(np.abs(g - r) / r)) for g, r in zip(sig_g, sig_r)],
        "sigma_abs_dev_over_s1": [float(np.max(np.abs(g - r)) / r[0]) for g, r in zip(sig_g, sig_r)],
        "sigma_oracle_head": [r[:4].tolist() for r in sig_r],
        "oracle_component_s": tm, "oracle_online_wall_s": wall,
        "host_cores": os.cpu_count(),
    }
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps(rep, indent=1))
    print(json.dumps({k: v for k, v in rep.items() if k != "oracle_component_s"}), flush=True)


if __name__ == "__main__":
    main()
