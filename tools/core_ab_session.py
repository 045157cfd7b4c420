"""Configuration-4 session event by event (r = 128, explicit basis): singular
values, basis orthonormality defect and Gauss-Newton counts after every
event, for the current core kernel or (ADROM_CORE_OLD=1, bisect build only)
the round-1 kernel.  Usage: core_ab_session.py <tag> <events>"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(os.environ.get("ADROM_ROOT", Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(ROOT))


def main(tag, n_events):
    import torch
    import bench
    from paper_2605_28684_b200.dense import ts_tn
    from paper_2605_28684_b200.driver import Session, offline_stage
    case = bench.rom_case("cfg4", 0)
    cfg, model = bench.rom_experiment(case)
    training, scaling, basis0 = offline_stage(cfg, model)
    q_last = training[cfg.w_init].clone()
    del training
    torch.cuda.empty_cache()
    sess = Session(cfg, model, adaptive=True)
    sess.load(scaling, basis0, q_last)
    sess.start()
    sig, defect, its = [], [], []
    err = ""
    for e in range(n_events):
        try:
            sess.advance(cfg.z)
        except Exception as exc:  # noqa: BLE001
            err = f"{type(exc).__name__}: {exc}"
            print("event", e, err, flush=True)
            break
        log, ev, a, s, _ = sess.read(cfg.z * (e + 1), e + 1)
        phi = sess.basis()
        g = ts_tn(phi, phi)
        d = float((g - torch.eye(g.shape[0], dtype=g.dtype, device=g.device)).abs().max())
        del phi, g
        sig.append(s.cpu().numpy())
        defect.append(d)
        its.append(log[-cfg.z:, 1].copy())
        print(f"event {e} defect {d:.3e} sig[-1] {sig[-1][-1]:.4e} its {its[-1].astype(int)} "
              f"ev_err {int(ev[-1].error)} resid {ev[-1].residual_norm:.4e}", flush=True)
    np.savez_compressed(ROOT / "gpurun_out" / f"c4ab_{tag}.npz", sig=np.array(sig), defect=np.array(defect),
                        its=np.array(its), err=np.array(err))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
