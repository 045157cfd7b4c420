"""cfg3 parity diagnostics with the QDEIM decisions separated from the
arithmetic: (1) the device loop's own sampled rows at selected events vs the
oracle's exact greedy and LAPACK geqp3 pivots on the SAME basis; (2) the
oracle loop re-run with the device loop's sampled rows pinned,
state deviation per step; (3) a nudged pinned oracle run (the envelope)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main(n=1 << 16, steps=200):
    import cfg3_parity as C
    from oracle import hyper
    setup = C.oracle_setup(n, steps)
    at = (1, 2, 5, 10, 20, 50, 100, 150, 200)
    got = C.gpu_run(setup, steps, keep_phi_at=at)
    print("gpu GN its mean", got["it"].mean(), "hist", np.bincount(got["it"]))
    for k in at:
        phi = got["phis"][k]
        g = np.array(hyper.greedy_pivots(phi, 64)[0])
        try:
            l = np.array(hyper.pivot_sequence(phi.T, 64))
        except Exception as e:  # noqa: BLE001
            l = np.array([-1])
        mine = got["samp"][k]
        first = next((j for j in range(64) if mine[j] != g[j]), None)
        print(f"event {k}: gpu==greedy {np.array_equal(mine, g)} (first diff {first}) "
              f"gpu==lapack(set) {np.array_equal(np.sort(mine), np.sort(l))} "
              f"greedy==lapack(set) {np.array_equal(np.sort(g), np.sort(l))}")
    pinned = [np.asarray(s, dtype=np.int64) for s in got["samp"]]
    ref_p = C.oracle_run(setup, steps, pinned=pinned)
    st = np.array(ref_p.states)
    dev = np.linalg.norm(got["traj"] - st, axis=1) / np.linalg.norm(st, axis=1)
    print("pinned: dev per 10 steps", np.array2string(dev[::10], precision=2))
    print("pinned: its equal", np.mean(np.array(ref_p.iterations) == got["it"]),
          "ref its mean", np.mean(ref_p.iterations))
    env = np.zeros(steps)
    for seed in (1, 2):
        e = C.oracle_run(setup, steps, pinned=pinned, nudge_seed=seed)
        env = np.maximum(env, np.linalg.norm(np.array(e.states) - st, axis=1) / np.linalg.norm(st, axis=1))
    print("pinned envelope per 10 steps", np.array2string(env[::10], precision=2))
    free = C.oracle_run(setup, steps)
    sf = np.array(free.states)
    print("free oracle vs pinned oracle per 10", np.array2string(
        np.linalg.norm(sf - st, axis=1)[::10] / np.linalg.norm(sf, axis=1)[::10], precision=2))
    print("free oracle its mean", np.mean(free.iterations), "norm growth", np.linalg.norm(sf[-1]) / np.linalg.norm(sf[0]),
          "gpu norm growth", np.linalg.norm(got["traj"][-1]) / np.linalg.norm(got["traj"][0]))


if __name__ == "__main__":
    main()
