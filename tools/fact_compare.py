"""Run the same session with the factored basis (ADROM_FACTORED=1) and the
explicit rotation (=0) and print the differences (diagnostics)."""
import os
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_28684_b200.driver import Session, offline_stage  # noqa: E402


def run(case_name, n, steps, fact):
    os.environ["ADROM_FACTORED"] = "1" if fact else "0"
    case = bench.rom_case(case_name, n)
    cfg, model = bench.rom_experiment(case)
    training, scaling, basis0 = offline_stage(cfg, model)
    sess = Session(cfg, model, adaptive=True)
    sess.load(scaling, basis0, training[cfg.w_init])
    sess.start()
    out = torch.empty((steps, model.n_dof), dtype=torch.float64, device="cuda")
    sess.advance(steps, 1, out, None)
    sess.finish()
    log, ev, a, sig, q = sess.read(steps, steps)
    idx = sess.sampling().cpu().numpy()
    phi = sess.basis()
    sess.close()
    return dict(traj=out.cpu().numpy(), log=log, ev=[(e.error, e.coarse_iterations) for e in ev],
                sig=sig.cpu().numpy(), idx=np.sort(idx), phi=phi)


for name, n, steps in [(a, int(b), int(c)) for a, b, c in (x.split(":") for x in sys.argv[1:])]:
    e = run(name, n, steps, False)
    f = run(name, n, steps, True)
    dev = np.linalg.norm(e["traj"] - f["traj"], axis=1) / np.linalg.norm(e["traj"], axis=1)
    print(f"== {name} N={n} steps={steps}")
    print("  traj rel dev: max %.3e last %.3e" % (dev.max(), dev[-1]))
    print("  sigma rel dev (first 8):", np.abs(e["sig"] - f["sig"])[:8] / e["sig"][:8])
    print("  sigma rel dev max over > 1e-8 s1: %.3e" % (np.max(np.abs(e["sig"] - f["sig"])[e["sig"] > 1e-8 * e["sig"][0]] / e["sig"][e["sig"] > 1e-8 * e["sig"][0]])))
    print("  iterations equal:", np.array_equal(e["log"][:, 1], f["log"][:, 1]),
          "events equal:", e["ev"] == f["ev"], "final idx equal:", np.array_equal(e["idx"], f["idx"]))
    pe, pf = e["phi"], f["phi"]
    g = pe.T @ pf
    u, s, vt = torch.linalg.svd(g)
    print("  basis: min cos of principal angles %.16f" % s.min().item())
