"""Where does the cfg3 e2e time go?  (diagnostics)"""
import sys, time
sys.path.insert(0, "/root/repo")
import torch
import bench
from paper_2605_28684_b200.driver import Session, offline_stage
from paper_2605_28684_b200.snapshots import ScalingTransform
from paper_2605_28684_b200.tracking import ReducedBasis
case = bench.rom_case("cfg3")
cfg, model = bench.rom_experiment(case)
K = 20
N = model.n_dof
training, scaling, basis0 = offline_stage(cfg, model)
pin = lambda x: x.detach().to("cpu").pin_memory()
h = dict(q_ref=pin(scaling.q_ref), d=pin(scaling.row_scale), phi=pin(basis0.phi), sig=pin(basis0.sigma), q_last=pin(training[cfg.w_init]))
phi_norm = scaling.phi_norm
del training, scaling, basis0
torch.cuda.empty_cache()
out = torch.empty((K, N), dtype=torch.float64, pin_memory=True)
for mode in ("host", "none", "host"):
    sess = Session(cfg, model, adaptive=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d = {k: v.to("cuda", non_blocking=True) for k, v in h.items()}
    torch.cuda.synchronize(); t1 = time.perf_counter()
    sess.load(ScalingTransform(q_ref=d["q_ref"], phi_norm=phi_norm), ReducedBasis(d["phi"], d["sig"]), d["q_last"])
    torch.cuda.synchronize(); t2 = time.perf_counter()
    sess.start()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    if mode == "host":
        sess.advance(K, 1, None, out)
    else:
        sess.advance(K)
    torch.cuda.synchronize(); t4 = time.perf_counter()
    sess.finish()
    torch.cuda.synchronize(); t5 = time.perf_counter()
    print(mode, "h2d %.1f load %.1f start %.1f advance %.1f (%.2f ms/step) finish %.1f total %.1f ms -> %.1f steps/s" % (
        1e3*(t1-t0), 1e3*(t2-t1), 1e3*(t3-t2), 1e3*(t4-t3), 1e3*(t4-t3)/K, 1e3*(t5-t4), 1e3*(t5-t0), K/(t5-t0)), flush=True)
    sess.close()
    del d
