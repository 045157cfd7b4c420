"""iSVD core SVD microbenchmark: isvd_update on a small N (the core kernel
dominates), r in {64, 128}; prints the core path and the per-call time.

    python tools/core_bench.py [--reps 50]
    ncu -k regex:isvd_core --set full python tools/core_bench.py --reps 3
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    import torch
    import paper_2605_28684_b200 as P
    for r in (64, 128):
        n = 4096
        rng = np.random.default_rng(r)
        phi = torch.from_numpy(np.linalg.qr(rng.standard_normal((n, r)))[0]).cuda()
        sig = torch.from_numpy(np.concatenate([np.logspace(0, -6, r // 2),
                                               1e-13 * (1 + 0.01 * np.arange(r - r // 2))])).cuda()
        y = torch.from_numpy(rng.standard_normal(n)).cuda()
        b = P.ReducedBasis(phi=phi, sigma=sig)
        P.isvd_update(b, y, 0.1, r)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(a.reps):
            P.isvd_update(b, y, 0.1, r)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / a.reps
        print(f"r={r}: {dt * 1e3:.3f} ms per isvd_update (N={n}); info={P.tracking.last_isvd_info()}")


if __name__ == "__main__":
    main()
