"""Time the coarse backward-Euler step (Newton + block-tridiagonal solve) at
cfg-3 size on device-resident state (diagnostics; not part of the bench)."""
import sys
import time

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

import paper_2605_28684_b200 as P  # noqa: E402
from paper_2605_28684_b200 import _lib  # noqa: E402
from paper_2605_28684_b200.configs import burgers_bump_ic  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
dt = float(sys.argv[2]) if len(sys.argv) > 2 else 1.4636781980260717e-08
m = P.BurgersProblem(n, nu=1e-3)
q = torch.from_numpy(burgers_bump_ic(n)).cuda()
ctx = _lib.Context.get()
for _ in range(3):
    res = P.implicit_step(m, q, dt)
torch.cuda.synchronize()
ctx.prof_enable(True)
t0 = time.perf_counter()
K = 10
for _ in range(K):
    res = P.implicit_step(m, q, dt)
torch.cuda.synchronize()
t1 = time.perf_counter()
print("implicit_step ms %.3f iterations %d" % ((t1 - t0) / K * 1e3, res.iterations))
print(ctx.prof_read())
