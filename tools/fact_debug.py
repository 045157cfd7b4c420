"""cfg3-shaped run in the factored mode: per-step QDEIM rounds, event errors."""
import sys
sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
from paper_2605_28684_b200 import _lib  # noqa: E402
from paper_2605_28684_b200.driver import Session, offline_stage  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 24
case = bench.rom_case("cfg3", n)
cfg, model = bench.rom_experiment(case)
training, scaling, basis0 = offline_stage(cfg, model)
sess = Session(cfg, model, adaptive=True)
sess.load(scaling, basis0, training[cfg.w_init])
ctx = _lib.Context.get()
sess.start()
ctx.prof_enable(True)
for k in range(steps):
    sess.advance(1)
    p = ctx.prof_read()
    q = p.get("qdeim_round", (0, 0))
    print("step", k, "qdeim rounds", q[1], "ms %.2f" % q[0], "resid %.3f" % p.get("isvd_resid", (0, 0))[0])
log, ev, *_ = sess.read(steps, steps)
print("events:", [(int(e.step), int(e.error)) for e in ev])
print(ctx.last_error() if hasattr(ctx, "last_error") else "")
