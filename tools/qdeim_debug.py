"""Print QDEIM verification passes per event and LSPG residual norms for a
cfg3-shaped run (diagnostics; not part of the bench)."""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import torch
import bench
from paper_2605_28684_b200 import _lib
from paper_2605_28684_b200.driver import Session, offline_stage
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
case = bench.rom_case("cfg3", n)
cfg, model = bench.rom_experiment(case)
training, scaling, basis0 = offline_stage(cfg, model)
sess = Session(cfg, model, adaptive=True)
sess.load(scaling, basis0, training[cfg.w_init])
ctx = _lib.Context.get()
sess.start()
ctx.prof_enable(True)
for k in range(6):
    sess.advance(1)
    p = ctx.prof_read()
    q = p.get("qdeim_round", (0, 0))
    print("step", k, "qdeim passes", q[1], "qdeim ms %.2f" % q[0], "rom", p.get("rom_step"))
log, ev, *_ = sess.read(6, 6)
print("rom log [conv, it, res]:", log.tolist())
