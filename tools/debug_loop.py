import sys, json, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2605_28684_b200 as P
from test_gpu_rom import _exp_config
from conftest import load_golden
for name in sys.argv[1:]:
    g = load_golden(name)
    cfg = _exp_config(name)
    res = P.run_adaptive_rom(cfg, truth=g["truth"])
    print(name, res.event_log[:3])
    traj = g["traj"][cfg.w_init + 1:]; got = res.trajectory[cfg.w_init + 1:]
    dev = np.linalg.norm(got - traj, axis=1) / np.linalg.norm(traj, axis=1)
    print("dev first/max", dev[:12], dev.max(), "env max", g["env_state"].max())
    print("iters ref", list(g["it"][:20])); print("iters got", list(res.step_iterations[:20]))
