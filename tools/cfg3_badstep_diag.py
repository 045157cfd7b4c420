"""Find the cfg3 (N=2^16) online steps where the device Gauss-Newton hits
max_iter, restart both the device session and the oracle from the device
loop's own state just before such a step (basis, sigma, decoded state), and
compare the first reduced step; the restart inputs are saved for offline
analysis (gpurun_out/cfg3_badstep_<k>.npz)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main(n=1 << 16, steps=200):
    import cfg3_parity as C
    from oracle import online
    setup = C.oracle_setup(n, steps)
    case, ocfg, training, q_ref, phi_norm, d, phi0, sigma0 = setup
    got = C.gpu_run(setup, steps)
    its = got["it"]
    bad = [k for k in range(1, steps) if its[k] >= 5][:4]      # 0-based step index k: step k+1
    print("gpu its >= 5 at online steps", [k + 1 for k in bad], "its", [int(its[k]) for k in bad])
    got2 = C.gpu_run(setup, steps, keep_phi_at=set(bad))        # basis after the event of step k
    for k in bad:
        phi_s = got2["phis"][k]
        sig_s = got2["sig"][k - 1]
        q_s = got2["traj"][k - 1]
        rec = online.run_online(ocfg, {case.w_init: q_s}, q_ref, d, phi_s, sig_s, keep_stride=1,
                                n_steps=2)
        sub = (case, ocfg, {case.w_init: q_s}, q_ref, phi_norm, d, phi_s, sig_s)
        g = C.gpu_run(sub, 2)
        dev = np.linalg.norm(g["traj"] - np.array(rec.states), axis=1) / np.linalg.norm(np.array(rec.states), axis=1)
        print(f"restart at step {k}: its gpu {g['it']} oracle {rec.iterations} dev {dev} "
              f"samp equal {[np.array_equal(np.sort(a), np.sort(b)) for a, b in zip(g['samp'], rec.samplings)]}")
        if k != bad[0]:
            continue  # one case travels back (gpurun_out <= 64 MiB)
        np.savez_compressed(ROOT / "gpurun_out" / f"cfg3_badstep_{k}.npz", phi=phi_s, sigma=sig_s, q=q_s,
                            its_gpu=g["it"], its_ref=np.array(rec.iterations), traj_gpu=g["traj"],
                            traj_ref=np.array(rec.states), a_ref=np.array(rec.reduced),
                            samp=np.array(rec.samplings[0]))


if __name__ == "__main__":
    main()
