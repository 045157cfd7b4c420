"""A/B of the iSVD core kernels at configuration 4's first event (r = 128,
explicit basis): the round-1 one-block Jacobi kernel (ADROM_CORE_OLD, only in
the bisect build) vs the current kernel, on the real offline basis and the
first coarse snapshot."""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(os.environ.get("ADROM_ROOT", Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(ROOT))


def main():
    import torch
    import bench
    import paper_2605_28684_b200 as P
    from paper_2605_28684_b200.driver import offline_stage
    from paper_2605_28684_b200.tracking import last_isvd_info
    case = bench.rom_case("cfg4", 0)
    cfg, model = bench.rom_experiment(case)
    training, scaling, basis0 = offline_stage(cfg, model)
    q_last = training[cfg.w_init].clone()
    del training
    torch.cuda.empty_cache()
    y = P.implicit_step(model, q_last, cfg.z * cfg.dt, cfg.stepper()).x
    yh = scaling.row_scale * (y - scaling.q_ref)
    out = {}
    for tag, old in (("new", None), ("old", "1")):
        if old:
            os.environ["ADROM_CORE_OLD"] = old
        else:
            os.environ.pop("ADROM_CORE_OLD", None)
        b = P.isvd_update(basis0, yh, cfg.rule.lam, cfg.r)
        info = last_isvd_info()
        out[tag] = (b.sigma.cpu().numpy(), b.phi[:, :].cpu().numpy()[:: 4096].copy(), info)
        print(tag, "info", info, "sigma[:3]", out[tag][0][:3], "sigma[-3:]", out[tag][0][-3:], flush=True)
        del b
        torch.cuda.empty_cache()
    sn, so = out["new"][0], out["old"][0]
    print("sigma rel max", np.max(np.abs(sn - so) / np.abs(so)), "abs/s1", np.max(np.abs(sn - so)) / so[0])
    pn, po = out["new"][1], out["old"][1]
    # column signs are arbitrary: align
    sg = np.sign(np.sum(pn * po, axis=0))
    print("phi sample max diff (sign aligned)", np.max(np.abs(pn * sg - po)), "per col worst",
          np.argsort(-np.max(np.abs(pn * sg - po), axis=0))[:8])
    print("sigma old", np.array2string(so, precision=3))


if __name__ == "__main__":
    main()
