"""Orthonormality defect of the configuration-3 session basis along the full
2000-step horizon (N = 2^24): max |Phi^T Phi - I| at a few steps, with the
singular values' head and tail."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import os
    import torch
    import bench
    from paper_2605_28684_b200.dense import ts_tn
    from paper_2605_28684_b200.driver import Session, offline_stage
    from paper_2605_28684_b200 import configs
    n_env = int(os.environ.get("ADROM_DEFECT_N", "0"))
    case = configs.cfg3(n_env) if n_env else bench.rom_case("cfg3", 0)  # the recipe on that grid
    cfg, model = bench.rom_experiment(case)
    training, scaling, basis0 = offline_stage(cfg, model)
    q_last = training[cfg.w_init].clone()
    del training
    torch.cuda.empty_cache()
    sess = Session(cfg, model, adaptive=True)
    sess.load(scaling, basis0, q_last)
    sess.start()
    done = 0
    for target in (100, 300, 600, 1000, 1400, 1800, 2000):
        sess.advance(target - done)
        done = target
        phi = sess.basis()
        g = ts_tn(phi, phi)
        d = float((g - torch.eye(g.shape[0], dtype=g.dtype, device=g.device)).abs().max())
        _, _, _, s, _ = sess.read(1, 1)
        s = s.cpu().numpy()
        print(f"step {target}: defect {d:.3e} sigma[0] {s[0]:.4e} sigma[4] {s[4]:.3e} sigma[-1] {s[-1]:.3e}",
              flush=True)
        del phi, g
    sess.close()


if __name__ == "__main__":
    main()
