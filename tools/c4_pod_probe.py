"""Probe: POD spectrum of the cfg4 offline window for a few (dt, w_init)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
from paper_2605_28684_b200.driver import offline_stage

for dt, w, npu in [(float(a), int(b), int(c)) for a, b, c in (x.split(',') for x in sys.argv[1:])]:
    case = bench.rom_case("cfg4").scaled(w_init=w)
    from dataclasses import replace
    case = replace(case, dt=dt, n_pulses=npu)
    cfg, model = bench.rom_experiment(case)
    t0 = time.time()
    try:
        tr, sc, b = offline_stage(cfg, model)
    except Exception as e:  # noqa: BLE001
        print(dt, w, "failed:", e, flush=True)
        continue
    s = b.sigma.cpu().numpy()
    phin = sc.phi_norm.cpu().numpy()
    print("  phi_norm", np.array2string(phin, precision=2), flush=True)
    print(dt, w, npu, f"{time.time()-t0:.1f}s", "s0 %.3e" % s[0], "s127/s0 %.3e" % (s[-1] / s[0]),
          "n>1e-8 %d n>1e-10 %d" % ((s > 1e-8 * s[0]).sum(), (s > 1e-10 * s[0]).sum()), flush=True)
    del tr, sc, b
    torch.cuda.empty_cache()
