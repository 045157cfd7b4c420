"""FOM residual kernels alone (adrom_rhs) at north-star sizes: GB/s against
the measured HBM copy peak.  Diagnostics for DESIGN.md §3 (not the bench)."""
import ctypes as C
import json
import sys

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

import paper_2605_28684_b200 as P  # noqa: E402
from paper_2605_28684_b200 import _lib  # noqa: E402
from paper_2605_28684_b200.configs import burgers_bump_ic  # noqa: E402

peak = json.load(open("/root/repo/MEASURED_PEAKS.json")).get("hbm_gbs", 6557.4)
ctx = _lib.Context.get()
cases = [("burgers", P.BurgersProblem(1 << 24, nu=1e-3), burgers_bump_ic(1 << 24), 16),
         ("sod", P.SodProblem(1 << 22), P.SodProblem(1 << 22).initial_state(), 48),
         ("reacting", P.ReactingEulerProblem(1 << 20), P.ReactingEulerProblem(1 << 20).initial_state(), 208)]
for name, m, q0, bpc in cases:
    q = torch.from_numpy(q0).cuda()
    out = torch.empty_like(q)
    mabi = m.abi()
    call = lambda: ctx.call("adrom_rhs", C.byref(mabi), _lib.ptr(q), _lib.ptr(out))  # noqa: E731
    for _ in range(5):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 50
    e0.record()
    for _ in range(K):
        call()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    gbs = bpc * m.n_elem / (ms * 1e-3) / 1e9
    print(json.dumps({"model": name, "n_elem": m.n_elem, "ms": round(ms, 4),
                      "gcells": round(m.n_elem / (ms * 1e-3) / 1e9, 2), "GB/s": round(gbs, 1),
                      "frac_of_measured_peak": round(gbs / peak, 3)}))
