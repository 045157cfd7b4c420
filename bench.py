#!/usr/bin/env python
"""Benchmark of the B200 adaptive-ROM hot path (driver contract, one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg3|cfg2|cfg1|cfg0]

Workloads (BASELINE.json configs; seeded synthetic inputs, no datasets):
  cfg3  Burgers N=2^24 adaptive ROM, iSVD every step (r=n_s=64)   [default]
        step = one online step of driver._run_rom (LSPG step + decode +
        coarse Newton + iSVD + QDEIM + operator rebuild + encode)
  cfg2  iSVD stream N=2^22, r=64: step = one rank-1 update (tracking.py:141)
  cfg1  Sod N=4096 adaptive ROM (LSPG + FGS, z=5)
  cfg0  Burgers N=1024 adaptive ROM (LSPG + QDEIM, z=10)

Multi-GPU: the path does not shard (replicas only); with N ranks
every rank runs an independent replica, `value` sums the replicas and the
time is the max over ranks (CUDA events, barrier + synchronize around the
timed region).

--impl reference times the CPU implementation of the same path (the oracle
port of the reference, oracle/; the reference itself is Python and does not
travel to the GPU box) on rank 0 with all host threads.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import re
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS = {}
try:
    PEAKS = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
except Exception:  # noqa: BLE001
    PEAKS = {}
HBM_PEAK = float(PEAKS.get("hbm_gbs", 6650.0))
HBM_PEAK_SRC = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in PEAKS else \
    "fallback 6.65 TB/s (B200_PROFILING.md)"
# FP64 tensor-core (DMMA m8n8k4) peak measured on this pool with
# tools/fp64_peak.cu (profiles/r1_fp64_peak.txt); MEASURED_PEAKS.json carries
# only HBM and bf16, and the whole path computes in fp64.
FP64_DMMA_PEAK = 37.0
FP64_DMMA_SRC = "measured FP64 DMMA peak (tools/fp64_peak.cu, profiles/r1_fp64_peak.txt)"


def ncu_traffic(kernel: str, workload: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed `ncu --set full` capture (profiles/traffic.json), if any."""
    try:
        t = json.loads((ROOT / "profiles" / "traffic.json").read_text())
        e = t.get(workload, {}).get(kernel)
        return e["bytes"] if e else None
    except Exception:  # noqa: BLE001
        return None


# --------------------------------------------------------------------------- utils

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "25"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self) -> dict:
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sms.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sms)}


def dist_setup():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64,
                     device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


def roofline(bytes_per_launch: float, ms_per_launch: float, traffic=None) -> dict:
    achieved = bytes_per_launch / (ms_per_launch * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": HBM_PEAK, "unit": "GB/s",
            "frac": round(achieved / HBM_PEAK, 4), "traffic": traffic, "peak_source": HBM_PEAK_SRC}


# --------------------------------------------------------------------------- cfg2

def cfg2_inputs(case, n_snap: int):
    """The seeded stream of configs.StreamCase (the recipe the parity tests
    use): the Gaussian and every snapshot's coefficients and noise come from
    numpy's default_rng streams on the host; the modes are the unique QR
    factor (positive R diagonal) of that Gaussian, computed on the device.
    Returns (n_snap, N) on the device: row k = snapshot k."""
    import torch
    g = torch.from_numpy(case.gaussian()).cuda()
    q, rr = torch.linalg.qr(g)
    del g
    q *= torch.where(torch.diagonal(rr) < 0, -1.0, 1.0)[None, :]
    coef = torch.from_numpy(np.stack([case.coefficients(k) for k in range(n_snap)], axis=1)).cuda()
    noise = torch.from_numpy(np.stack([case.noise_vector(k) for k in range(n_snap)], axis=0)).cuda()
    snaps = (q @ coef).T.contiguous()
    snaps += case.noise * noise
    del q, noise
    return snaps


def bench_cfg2(args, rank, world):
    import ctypes as C
    import torch
    from paper_2605_28684_b200 import _lib
    from paper_2605_28684_b200.configs import cfg2
    case = cfg2()
    if args.n:
        case = type(case)(n=args.n)
    n, r = case.n, case.r
    K, W = args.steps, args.warmup
    snaps = cfg2_inputs(case, r + W + K)
    # setup (untimed): thin_svd of the first r snapshots (device Householder
    # QR + Jacobi SVD; the column signs are immaterial to the stream)
    from paper_2605_28684_b200.snapshots import pod
    b0 = pod(snaps[:r].T.contiguous(), r)
    phi, sig = b0.phi, b0.sigma
    ctx = _lib.Context.get()
    P = _lib.ptr
    # the streaming form (factored basis, csrc/factored.cu): every update is
    # tracking.py:141-178; the basis is materialised after the timed region
    from paper_2605_28684_b200.tracking import IsvdStream, ReducedBasis
    stream = IsvdStream(ReducedBasis(phi=phi, sigma=sig))

    def update(k):
        stream.update(snaps[r + k], case.lam)

    for k in range(W):
        update(k)
    torch.cuda.synchronize()
    barrier(world)
    ctx.prof_enable(True)
    l0 = ctx.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        ev0.record()
        for k in range(W, W + K):
            update(k)
        ev1.record()
        torch.cuda.synchronize()
    launches = ctx.launches() - l0
    probes = ctx.prof_read()
    ctx.prof_enable(False)
    ms = ev0.elapsed_time(ev1)
    ms = max_over_ranks(ms, world)
    barrier(world)
    ms_step = ms / K
    value = world * K / (ms * 1e-3)
    # pass 1 of the stream is HBM bound: 8 N (r + k + 1) bytes (A, the k live
    # residual columns, y), k cycling 0..15 between re-anchors
    kq = 16
    k_mean = float(np.mean([j % kq for j in range(W, W + K)]))
    p1_ms, p1_n = probes.get("isvd_project", (0.0, 0))
    p1_bytes = 8.0 * n * (r + k_mean + 1)
    canon = 8.0 * (3 * n * r + 2 * n)
    basis_out = stream.basis()
    phi, sig = basis_out.phi, basis_out.sigma
    stream.close()
    extra = {
        "isvd_update_ms": round(ms_step, 4),
        "isvd_update_hbm_frac": round(canon / (ms_step * 1e-3) / 1e9 / HBM_PEAK, 4),
        "isvd_update_canonical_bytes": canon,
        "probes_ms": {k: round(v[0] / max(v[1], 1), 4) for k, v in probes.items()},
        "reorth_passes": probes.get("isvd_resid", (0, 0))[1],
    }
    line = {
        "metric": "iSVD rank-1 updates/s (N=2^22, r=64); iSVD % of HBM roofline",
        "value": round(value, 3), "unit": "updates/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (configs.StreamCase: seeded rank-96 stream, numpy default_rng)",
        "config": {"workload": "cfg2-isvd-stream", "n": n, "r": r, "lam": case.lam,
                   "l2": "inputs larger than L2 (basis 2 GiB)", "parallelism": f"replicas{world}"},
        "roofline": roofline(p1_bytes, p1_ms / max(p1_n, 1)) if p1_n else None,
        "gpu_launches": launches,
    }
    if line["roofline"]:
        line["roofline"].update({"kernel": "isvd_project (xpass_kernel<64,1>: X^T y, factored basis)",
                                 "work_per_launch": {"bytes": p1_bytes, "k_mean": k_mean}})
    line.update(extra)
    line["clocks"] = clk.summary()
    if rank == 0 and not args.no_e2e:
        line["e2e"] = e2e_cfg2(args, case, snaps, phi, sig)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_cfg2(case)
    if rank == 0 and not args.n:
        line["batch_svd_diag"] = cfg2_batch_diag()
    return line


def cfg2_batch_diag(n=1 << 14, updates=10000):
    """BASELINE configs[2]'s check "largest principal angle against a batch
    SVD of all snapshots" (a diagnostic: truncated iSVD on
    rank-96 data is not the batch SVD).  The full 10,000-update stream of the
    seeded recipe at N = 2^14 (a batch SVD of the 2^22 x 10,064 matrix is
    337 GB): the device iSVD stream vs the top-64 left singular subspace of
    all snapshots (eigenvectors of the snapshot Gram X^T X, lifted by X;
    computed with torch as an untimed diagnostic), sine-based angle."""
    import torch
    from paper_2605_28684_b200.configs import StreamCase
    from paper_2605_28684_b200.dense import max_principal_angle
    from paper_2605_28684_b200.snapshots import pod
    from paper_2605_28684_b200.tracking import IsvdStream, ReducedBasis
    t0 = time.perf_counter()
    case = StreamCase(n=n, updates=updates)
    r = case.r
    x = cfg2_inputs(case, r + updates)                 # (r + updates) x n on the device
    b0 = pod(x[:r].T.contiguous(), r)                  # thin_svd of x_0 .. x_{r-1}
    stream = IsvdStream(ReducedBasis(phi=b0.phi, sigma=b0.sigma))
    for k in range(updates):
        stream.update(x[r + k], case.lam)
    got = stream.basis()
    stream.close()
    g = x @ x.T                                        # snapshot Gram (m x m)
    ev, vec = torch.linalg.eigh(g)
    top = torch.argsort(ev, descending=True)[:r]
    sb = ev[top].clamp(min=0).sqrt()
    ub = (x.T @ vec[:, top]) / sb[None, :]
    ang = max_principal_angle(ub, got.phi)
    sg = got.sigma
    return {"n": n, "updates": updates, "lam": case.lam,
            "max_principal_angle_rad": float(ang),
            "sigma_rel_dev_max": float(((sg - sb).abs() / sb).max()),
            "sigma1_isvd": float(sg[0]), "sigma1_batch": float(sb[0]),
            "sigma64_isvd": float(sg[-1]), "sigma64_batch": float(sb[-1]),
            "seconds": round(time.perf_counter() - t0, 1),
            "note": "diagnostic only: truncation to r=64 of a rank-96 stream departs from the batch "
                    "SVD by design (SURVEY §8c-6); the parity gate is iSVD vs the CPU isvd_update"}


def e2e_cfg2(args, case, snaps, phi, sig):
    """The streaming update through the public API (tracking.IsvdStream) with
    HOST buffers: every step copies its snapshot from pinned host memory and
    reads the step's result (the singular values) back; the basis is state
    and stays on the device (materialised by IsvdStream.basis() on demand)."""
    import torch
    from paper_2605_28684_b200.tracking import IsvdStream, ReducedBasis
    n, r = case.n, case.r
    steps = args.steps
    h_y = torch.empty((steps, n), dtype=torch.float64, pin_memory=True)
    h_y.copy_(snaps[-steps:])
    h_sig = torch.empty((steps, r), dtype=torch.float64, pin_memory=True)
    # snapshot k+1 crosses the host link on a copy stream while update k runs
    # (two device slots; each update returns only after its kernels, so the
    # slot it read is free when the copy after next lands in it)
    d_y = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(2)]
    copy_stream = torch.cuda.Stream()
    stream = IsvdStream(ReducedBasis(phi=phi, sigma=sig))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(copy_stream):
        d_y[0].copy_(h_y[0], non_blocking=True)
        ready[0].record(copy_stream)
    for k in range(steps):
        cur = k & 1
        torch.cuda.current_stream().wait_event(ready[cur])
        if k + 1 < steps:
            with torch.cuda.stream(copy_stream):
                d_y[1 - cur].copy_(h_y[k + 1], non_blocking=True)
                ready[1 - cur].record(copy_stream)
        stream.update(d_y[cur], case.lam)
        h_sig[k].copy_(stream.basis_sigma(), non_blocking=True)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / steps
    stream.close()
    return {"value": round(1e3 / ms, 3), "unit": "updates/s", "ms_per_step": round(ms, 3),
            "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * r, "steps": steps,
            "note": "IsvdStream: snapshot H2D (double-buffered on a copy stream) + singular values "
                    "D2H per update; wall clock"}


def cpu_baseline_cfg2(case, n_sample=0, reps=2):
    """Oracle port of tracking.isvd_update (gelsd least squares, as the
    reference) on the host, timed AT THE BENCHMARKED N (a bounded sample of
    `reps` updates, ~8 s each at N = 2^22)."""
    from oracle import subspace
    rng = np.random.default_rng(0)
    r = case.r
    n_sample = n_sample or case.n
    phi = np.linalg.qr(rng.standard_normal((n_sample, r)))[0]
    sig = np.linspace(10, 1, r)
    ys = [rng.standard_normal(n_sample) for _ in range(reps)]
    t0 = time.perf_counter()
    for y in ys:
        phi, sig, _ = subspace.isvd_update(phi, sig, y, case.lam, r)
    dt = (time.perf_counter() - t0) / reps
    scale = n_sample / case.n
    return {"value": round(scale / dt, 6), "unit": "updates/s", "cores": cpu_cores(),
            "kind": "port", "same_config": n_sample == case.n,
            "sample": f"{reps} oracle isvd_update (numpy/LAPACK gelsd) at N={n_sample}, r={r}: "
                      f"{dt:.2f} s/update" + ("" if n_sample == case.n else
                                              f", scaled x{case.n // n_sample} to N={case.n}")}


def reference_cfg2(args, rank, world):
    if rank != 0:
        return None
    from paper_2605_28684_b200.configs import cfg2
    case = cfg2()
    if args.n:
        case = type(case)(n=args.n)
    # the benchmarked N; an update is ~8 s of gelsd at N = 2^22, so the timed
    # sample is bounded to 3 updates after 1 warm-up (the line says so)
    n_sample = case.n
    n_warm, n_timed = min(args.warmup, 1), max(1, min(args.steps, 3))
    from oracle import subspace
    rng = np.random.default_rng(1)
    r = case.r
    phi = np.linalg.qr(rng.standard_normal((n_sample, r)))[0]
    sig = np.linspace(10, 1, r)
    for _ in range(n_warm):
        phi, sig, _ = subspace.isvd_update(phi, sig, rng.standard_normal(n_sample), case.lam, r)
    ys = [rng.standard_normal(n_sample) for _ in range(n_timed)]
    t0 = time.perf_counter()
    for y in ys:
        phi, sig, _ = subspace.isvd_update(phi, sig, y, case.lam, r)
    dt = (time.perf_counter() - t0) / n_timed
    value = 1.0 / dt
    return {
        "metric": "iSVD rank-1 updates/s (N=2^22, r=64); iSVD % of HBM roofline",
        "impl": "reference", "value": round(value, 6), "unit": "updates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 / value, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": "cfg2-isvd-stream", "n": case.n, "r": r},
        "cpu_baseline": {"value": round(value, 6), "unit": "updates/s", "cores": cpu_cores(),
                         "kind": "port", "same_config": True,
                         "sample": f"{n_timed} oracle isvd_update (gelsd) at N={n_sample} after "
                                   f"{n_warm} warm-up (bounded sample of the {args.steps} steps asked)"},
        "e2e": {"value": round(value, 6), "unit": "updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


# --------------------------------------------------------------------------- ROM loops

def rom_case(name: str, n_override: int = 0):
    from paper_2605_28684_b200 import configs
    case = {"cfg0": configs.cfg0, "cfg1": configs.cfg1, "cfg3": configs.cfg3,
            "cfg4": configs.cfg4}[name]()
    if n_override:
        case = case.scaled(n_elem=n_override)
    return case


def rom_experiment(case):
    import paper_2605_28684_b200 as P
    cfg = P.ExperimentConfig(
        model=case.model, n_elem=case.n_elem, nu=case.nu, gamma=case.gamma, dt=case.dt,
        n_t=case.n_t, w_init=case.w_init, r=case.r, n_s=case.n_s, z=case.z,
        rule=P.UpdateRule("isvd", lam=case.lam), projection=case.projection,
        sampling=case.sampling, feature=case.feature, n_extra=case.n_extra)
    ic = case.initial_state()
    if case.model == "reacting":  # configuration 4: the seeded pulse IC is the model's own
        return cfg, P.ReactingEulerProblem(case.n_elem, gamma=case.gamma, n_pulses=case.n_pulses)
    base = P.BurgersProblem if case.model == "burgers" else P.SodProblem

    class Problem(base):  # the seeded IC of the case (driver.make_problem + custom IC)
        def initial_state(self):
            return ic.copy()

    model = Problem(case.n_elem, nu=case.nu) if case.model == "burgers" else Problem(case.n_elem)
    return cfg, model


ROM_METRIC = "adaptive-ROM online steps/s; FOM residual Gcell/s and iSVD % of HBM roofline"


def residual_alone(model, q):
    """The FOM residual kernel (adrom_rhs) timed alone on
    the device on the run's state: inside the loop it runs on the coarse-step
    stream at low priority, overlapped with the reduced step, so its probe
    time there is not a kernel time.  16 n_var bytes per cell."""
    import ctypes as C
    import torch
    from paper_2605_28684_b200 import _lib
    ctx = _lib.Context.get()
    out = torch.empty_like(q)
    mabi = model.abi()
    call = lambda: ctx.call("adrom_rhs", C.byref(mabi), _lib.ptr(q), _lib.ptr(out))  # noqa: E731
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    bpc = 16.0 * model.n_var
    gbs = bpc * model.n_elem / (ms * 1e-3) / 1e9
    return {"gcells": round(model.n_elem / (ms * 1e-3) / 1e9, 2), "ms": round(ms, 4),
            "GB/s": round(gbs, 1), "hbm_frac": round(gbs / HBM_PEAK, 4),
            "bytes_per_cell": bpc, "kernel": "adrom_rhs alone (CUDA events, input > L2)"
            if 2 * 8 * model.n_dof > 126e6 else "adrom_rhs alone (CUDA events, L2-resident)"}


def bench_rom(args, rank, world):
    import torch
    from paper_2605_28684_b200 import _lib
    from paper_2605_28684_b200.driver import Session, offline_stage
    from paper_2605_28684_b200.errors import RomStepError
    case = rom_case(args.config, args.n)
    cfg, model = rom_experiment(case)
    K, W = args.steps, args.warmup
    N, r = model.n_dof, case.r
    if W + K > case.n_t - case.w_init:
        raise SystemExit("steps + warmup exceed the online horizon")
    t_off = time.perf_counter()
    training, scaling, basis0 = offline_stage(cfg, model)
    q_last = training[cfg.w_init].clone()
    del training
    torch.cuda.synchronize()
    torch.cuda.empty_cache()  # the offline window (17 GB at cfg4) leaves torch's cache
    t_off = time.perf_counter() - t_off
    ctx = _lib.Context.get()
    sess = Session(cfg, model, adaptive=True)
    sess.load(scaling, basis0, q_last)
    t0 = time.perf_counter()
    sess.start()  # driver.py:321-331 (first lookahead + sampling without pivot guesses)
    torch.cuda.synchronize()
    t_start = time.perf_counter() - t0
    sess.advance(W)
    torch.cuda.synchronize()
    barrier(world)
    l0 = ctx.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prof_timed = os.environ.get("ADROM_PROFILE_TIMED") == "1"  # ncu --profile-from-start off
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        if prof_timed:
            torch.cuda.cudart().cudaProfilerStart()
        ev0.record()
        sess.advance(K)
        ev1.record()
        torch.cuda.synchronize()
        if prof_timed:
            torch.cuda.cudart().cudaProfilerStop()
    launches = ctx.launches() - l0
    ms = max_over_ranks(ev0.elapsed_time(ev1), world)
    # kernel breakdown: the same number of further steps with the CUDA-event
    # probes on (they add a record pair per probe, so the timed region above
    # runs without them); shares are relative to this probed stretch
    kp = min(K, case.n_t - case.w_init - W - K)
    ctx.prof_enable(True)
    ep0, ep1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ep0.record()
    probed_note = None
    if kp > 0:
        try:
            sess.advance(kp)
        except RomStepError as exc:
            # the reference aborts a run whose reduced step fails (driver.py:338);
            # the probes recorded up to there still give the kernel shares
            probed_note = f"probed stretch aborted like the reference would: {exc}"
    ep1.record()
    torch.cuda.synchronize()
    probes = ctx.prof_read()
    ctx.prof_enable(False)
    ms_probed = ep0.elapsed_time(ep1) if kp > 0 else ms
    log, events, *_ = sess.read(W + K, W + K)
    sess.close()
    barrier(world)
    ms_step = ms / K
    value = world * K / (ms * 1e-3)
    per = {k: (v[0] / max(v[1], 1), v[1]) for k, v in probes.items()}
    share = {k: round(v[0] / ms_probed, 4) for k, v in probes.items()}
    # Roofline.  Explicit basis (r not in {32, 64} or small N): the iSVD
    # rotation Phi' = [Phi | q_hat] B (rot_tc_kernel, FP64 DMMA), 2 N r (r+1)
    # flop.  Factored basis (csrc/factored.cu, the cfg-3 path): no rotation;
    # the largest single kernel is the first basis pass (xpass_tma_kernel
    # MODE 1: X^T y and exact row norms, tiles staged by the copy engine),
    # HBM bound with algorithmic bytes 8 N (r + k + 3): A, the k live
    # residual columns, y, and the row-norm read + write.  k cycles 0..15
    # between re-anchors (one event per step here); the mean over the timed
    # events is used.  QDEIM is larger in total but is a sequence of rounds of small
    # kernels (qdeim_rounds_per_step below).
    roof = roof1 = None
    if case.model == "reacting" and "decode" in per:
        # configuration 4: the largest kernels are FP64-pipe bound (the FD
        # directions of the large-sample LSPG step, bl_dir_kernel, ~1.4 ms per
        # Gauss-Newton iteration; the coarse step's 13x13 block solve on the
        # tensor cores).  The HBM roofline is reported on the per-step decode
        # q~ = q_ref + (Phi a) / d (stream_kernel<128>: Phi read, q_ref and d
        # read, q~ written: 8 N (r + 3) bytes)
        dbytes = 8.0 * N * (r + 3)
        roof = roofline(dbytes, per["decode"][0], ncu_traffic("stream_kernel<128, 1, 1, 0>", case.name))
        roof.update({"kernel": "decode (stream_kernel<128>: q_ref + Phi a / d)",
                     "work_per_launch": {"bytes": dbytes},
                     "share_of_step": round(probes["decode"][0] / ms_probed, 4),
                     "dominant_kernel": {"name": "bl_dir_kernel<reacting> (FD directions, FP64 pipe)",
                                         "share_of_step": round(probes.get("rom_step", (0, 0))[0] / ms_probed, 4),
                                         "note": "rom_step share; ncu: FP64 pipe 24 % active, "
                                                 "profiles/r1_cfg4_lspg_kernels_full.txt"}})
    elif "isvd_rotate" in per:
        rot_ms = per["isvd_rotate"][0]
        flops = 2.0 * N * r * (r + 1)
        rbytes = 8.0 * (2 * N * r + N) + 8.0 * 5 * N + 1.0 * N
        tf = flops / (rot_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": round(tf, 2), "peak": FP64_DMMA_PEAK,
                "unit": "TFLOP/s", "frac": round(tf / FP64_DMMA_PEAK, 4),
                "traffic": ncu_traffic("rot_tc_kernel<64>", case.name), "peak_source": FP64_DMMA_SRC,
                "kernel": "isvd_rotate (rot_tc_kernel, FP64 DMMA)",
                "work_per_launch": {"flops": flops, "bytes": rbytes},
                "hbm_achieved_gbs": round(rbytes / (rot_ms * 1e-3) / 1e9, 1),
                "hbm_frac": round(rbytes / (rot_ms * 1e-3) / 1e9 / HBM_PEAK, 4),
                "share_of_step": round(probes["isvd_rotate"][0] / ms_probed, 4)}
    elif "isvd_project" in per:
        kq = 16
        k_mean = float(np.mean([(j % kq) for j in range(W + K, W + K + max(kp, 1))])) if case.z == 1 else 0.0
        # the largest single kernel of the step (serialised launch list,
        # profiles/r2_cfg3_timed_launches.txt) is pass 2 (q = y - X(Wp) into
        # its Q panel, X^T q, state-transfer sums, fused decode): reads A, the
        # k live Q columns, y, q_ref, d; writes q and q~: 8 N (r + k + 5)
        x2bytes = 8.0 * N * (r + k_mean + 5)
        roof = roofline(x2bytes, per["isvd_resid"][0],
                        ncu_traffic("xpass_tma_kernel<64, 2>", case.name))
        roof.update({"kernel": "isvd_resid (xpass_tma_kernel<64,2>: q = y - X(Wp), X^T q, "
                               "state-transfer sums, fused decode; TMA-staged row tiles)",
                     "work_per_launch": {"bytes": x2bytes, "k_mean": k_mean},
                     "share_of_step": round(probes["isvd_resid"][0] / ms_probed, 4)})
        # pass 1 (X^T y + exact row norms): 8 N (r + k + 3)
        xbytes = 8.0 * N * (r + k_mean + 3)
        roof1 = roofline(xbytes, per["isvd_project"][0],
                         ncu_traffic("xpass_tma_kernel<64, 1>", case.name))
        roof1.update({"kernel": "isvd_project (xpass_tma_kernel<64,1>)",
                      "work_per_launch": {"bytes": xbytes, "k_mean": k_mean},
                      "share_of_step": round(probes["isvd_project"][0] / ms_probed, 4)})
    isvd_keys = ("isvd_project", "isvd_resid", "isvd_core", "isvd_rotate")
    n_upd = max(probes.get("isvd_project", (0, 1))[1], 1)
    isvd_ms = sum(probes.get(k, (0, 0))[0] for k in isvd_keys) / n_upd
    canon = 8.0 * (3 * N * r + 2 * N)
    fres = residual_alone(model, q_last)
    line = {
        "metric": ROM_METRIC, "value": round(value, 3), "unit": "online steps/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": {"burgers": "synthetic (seeded Burgers bump IC, configs.py)",
                 "sod": "synthetic (Sod Riemann data)",
                 "reacting": "synthetic (seeded mechanism and pulse IC, DESIGN.md §9)"}[case.model],
        "config": {"workload": case.name, "n_elem": case.n_elem, "r": r, "n_s": case.n_s,
                   "z": case.z, "lam": case.lam, "dt": case.dt, "projection": case.projection,
                   "sampling": case.sampling,
                   "l2": "inputs larger than L2 (basis %.1f GB)" % (8 * N * r / 1e9)
                         if 8 * N * r > 126e6 else "working set L2-resident (latency-bound)",
                   "parallelism": f"replicas{world}"},
        "roofline": roof,
        "roofline_pass1": roof1 if "isvd_project" in per and "isvd_rotate" not in per
                          and case.model != "reacting" else None,
        "gpu_launches": launches,
        "fom_residual_gcells": fres["gcells"],
        "fom_residual": fres,
        "isvd_update_ms": round(isvd_ms, 4),
        # canonical bytes of one update (2 reads + 1 write of Phi) over the
        # measured update time; the factored basis skips the write, so this
        # "fraction of the canonical roofline" can approach or pass 1
        "isvd_update_hbm_frac": round(canon / (isvd_ms * 1e-3) / 1e9 / HBM_PEAK, 4) if isvd_ms else None,
        "isvd_basis": "factored" if "isvd_rotate" not in per else "explicit",
        "probes_ms_per_launch": {k: round(v[0], 4) for k, v in per.items()},
        "probes_launches": {k: v[1] for k, v in per.items()},
        "share_of_step": share,
        "setup_s": {"offline": round(t_off, 3), "start": round(t_start, 3)},
        "rom_iterations_mean": float(np.mean(log[:, 1])) if len(log) else None,
        "qdeim_rounds_per_step": round(probes.get("qdeim_round", (0, 0))[1] / max(kp, 1), 2),
        "probed_steps": {"steps": kp, "aborted": probed_note,
                         "ms_per_step": round(ms_probed / max(kp, 1), 4),
                         "note": "kernel breakdown from a second stretch with CUDA-event probes on; "
                                 "the timed region runs without them"},
        "event_errors": sum(1 for e in events if e.error),
    }
    line["clocks"] = clk.summary()
    if rank == 0 and not args.no_e2e:
        line["e2e"] = e2e_rom(args, case)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_rom(case)
    return line


E2E_MIN_STEPS = 200
E2E_RING = 8


def e2e_rom(args, case):
    """Online loop through the C-ABI session with HOST buffers: the offline
    results (basis, scaling, last training state) are copied in from pinned
    host memory inside the timed region, and every step's decoded state is
    copied back to pinned host memory (the reference keeps its trajectory on
    the host, driver.py:306/344) — into a ring of E2E_RING host slots, since a
    full trajectory of 2^24-cell states does not fit in pinned memory.  The
    horizon is the reference's whole timed region (driver.py:319-389: all
    n_t - w_init online steps; --e2e-steps overrides), so the one-time upload
    of the offline basis (8.6 GB at cfg 3) is amortised like the reference's
    setup is."""
    import torch
    from paper_2605_28684_b200.driver import Session, offline_stage
    from paper_2605_28684_b200.errors import RomStepError
    cfg, model = rom_experiment(case)
    # the reference's timed region covers every online step (driver.py:319-389)
    K = min(case.n_t - case.w_init, max(args.steps, args.e2e_steps or (case.n_t - case.w_init)))
    if case.model == "reacting":
        # configuration 4's synthetic ROM degenerates after its second event
        # (the Gauss-Newton solve stops converging and the reduced Jacobian's
        # condition number reaches the reference's 1e14 RomStepError bound
        # around online step 26): the e2e horizon is the device-timed one
        K = min(K, args.warmup + args.steps)
    N, r = model.n_dof, case.r
    training, scaling, basis0 = offline_stage(cfg, model)
    pin = lambda x: x.detach().to("cpu").pin_memory()  # noqa: E731
    h = dict(q_ref=pin(scaling.q_ref), d=pin(scaling.row_scale), phi=pin(basis0.phi),
             sig=pin(basis0.sigma), q_last=pin(training[cfg.w_init]))
    phi_norm = scaling.phi_norm
    del training, scaling, basis0
    torch.cuda.empty_cache()
    out = torch.empty((E2E_RING, N), dtype=torch.float64, pin_memory=True)
    sess = Session(cfg, model, adaptive=True)
    sess.set_host_ring(E2E_RING)
    from paper_2605_28684_b200.snapshots import ScalingTransform
    from paper_2605_28684_b200.tracking import ReducedBasis
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d = {k: v.to("cuda", non_blocking=True) for k, v in h.items()}
    sess.load(ScalingTransform(q_ref=d["q_ref"], phi_norm=phi_norm), ReducedBasis(d["phi"], d["sig"]),
              d["q_last"])
    sess.start()
    try:
        sess.advance(K, 1, None, out)
        sess.finish()
    except RomStepError as exc:
        # The reduced step failed inside the horizon (rank-deficient sampled
        # Jacobian): the reference aborts such a run (driver.py:338), and its
        # own algorithm does on this workload too (configuration 1: the oracle
        # stops at online step 450).  Measure the horizon
        # that completes instead.
        sess.close()
        m = re.search(r"online step (\d+)", str(exc))
        k_ok = (int(m.group(1)) - case.w_init - 2) if m else 0
        if k_ok < 1 or getattr(args, "_e2e_retry", False):
            return {"value": None, "unit": "online steps/s", "steps": 0, "aborted": str(exc)}
        args2 = argparse.Namespace(**vars(args))
        args2.e2e_steps, args2.steps, args2._e2e_retry = k_ok, min(args.steps, k_ok), True
        res = e2e_rom(args2, case)
        res["horizon_cut"] = f"{exc}; e2e measured over the {k_ok} steps before it"
        return res
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    sess.close()
    h2d = sum(v.numel() * 8 for v in h.values())
    return {"value": round(K / wall, 3), "unit": "online steps/s", "steps": K,
            "h2d_bytes_per_step": int(h2d / K), "d2h_bytes_per_step": 8 * N,
            "note": f"timed region = reference's (driver.py:319-389) incl. start, over {K} online "
                    f"steps, plus the H2D of the offline results ({h2d / 1e9:.2f} GB once) and a "
                    f"D2H of every decoded state into pinned host memory "
                    f"({E2E_RING}-slot ring); wall clock"}


def _oracle_loop_config(case, n_elem, steps):
    from oracle import online, physics
    if case.model == "reacting":
        from oracle import reacting as R
        n_s = math.ceil(0.03 * n_elem) * 13
        small = case.scaled(n_elem=n_elem, n_s=n_s, n_extra=n_s - case.r)
        m = physics.Model("reacting", n_elem, gamma=small.gamma, mech=tuple(R.mechanism().ravel()))
    else:
        small = case.scaled(n_elem=n_elem)
        m = physics.Model(small.model, n_elem, nu=small.nu, gamma=small.gamma)
    ocfg = online.LoopConfig(model=m, dt=small.dt, n_t=small.w_init + steps + 1, w_init=small.w_init,
                             r=small.r, n_s=small.n_s, z=small.z, lam=small.lam,
                             projection=small.projection, sampling=small.sampling,
                             feature=small.feature, n_extra=small.n_extra)
    return small, ocfg


def cpu_loop_rom(case, steps):
    """The oracle's restatement of driver._run_rom (numpy/scipy: gelsd iSVD,
    geqp3 QDEIM, banded-LU Newton) on the host cores AT THE CASE'S OWN GRID:
    the start (driver.py:319-331) and `steps` online steps timed separately,
    per-step cost = steps' time / steps + start / n_online (the reference's
    timed region amortises its start over the whole horizon)."""
    from oracle import online
    small, ocfg = _oracle_loop_config(case, case.n_elem, steps)
    training = online.training_states(ocfg, small.initial_state())
    q_ref, d, phi0, sigma0 = online.offline(ocfg, training)
    online.run_online(ocfg, training, q_ref, d, phi0, sigma0, keep_stride=10 ** 9, n_steps=0)  # warm-up
    t0 = time.perf_counter()
    online.run_online(ocfg, training, q_ref, d, phi0, sigma0, keep_stride=10 ** 9, n_steps=0)
    t_start = time.perf_counter() - t0
    t0 = time.perf_counter()
    online.run_online(ocfg, training, q_ref, d, phi0, sigma0, keep_stride=10 ** 9, n_steps=steps)
    t_all = time.perf_counter() - t0
    n_online = case.n_t - case.w_init
    per_step = max(t_all - t_start, 1e-9) / steps + t_start / n_online
    return per_step, {"start_s": round(t_start, 4), "steps_s": round(t_all - t_start, 4),
                      "sample": f"oracle online loop at N={case.n_elem} (the benchmarked grid): "
                                f"start {t_start:.3f} s + {steps} steps {t_all - t_start:.3f} s, "
                                f"start amortised over {n_online} online steps"}


def cpu_step_full_grid(case):
    """One online step of driver._run_rom (driver.py:337-387) at the full
    grid (configuration 3: N = 2^24, r = n_s = 64) on the host cores, every
    component run once by the oracle's restatement of the reference
    (numpy/scipy: gelsd iSVD, geqp3 QDEIM, banded Newton, numpy residual,
    encode/decode): a bounded sample of ~2 minutes.

    The offline results are synthetic stand-ins with the real shapes: the
    reference's training window (64 backward-Euler steps at 2^24 cells, ~8
    min on the host) is replaced by q_ref = q_last = the seeded IC, D = 1
    (n_var = 1: driver.py:232-247) and an orthonormal Fourier basis with
    geometric singular values; the initial sampling is a fixed row set.
    The timed components cost the same for any input of these shapes
    (LAPACK gelsd / geqp3 and the residual passes are data-independent;
    the coarse step takes one Newton iteration at this dt either way).
    Returns (seconds per online step with the start amortised, detail)."""
    from oracle import hyper, online, physics, reduced, subspace
    n, r = case.n_elem, case.r
    u0 = case.initial_state()
    x = (np.arange(n) + 0.5) / n
    phi = np.empty((n, r))
    for j in range(r):
        w = 2.0 * np.pi * (j // 2 + 1) * x
        phi[:, j] = np.sqrt(2.0 / n) * (np.cos(w) if j % 2 == 0 else np.sin(w))
    sigma = 0.5 ** np.arange(r, dtype=float)
    q_ref = u0.copy()
    d = np.ones(n)
    m = physics.Model("burgers", n, nu=case.nu)
    ocfg = online.LoopConfig(model=m, dt=case.dt, n_t=case.n_t, w_init=case.w_init, r=r,
                             n_s=case.n_s, z=case.z, lam=case.lam)
    idx = np.sort(np.random.default_rng(0).choice(n, case.n_s, replace=False)).astype(np.int64)
    samp = hyper.closure(hyper.Sampling(indices=idx, closure=np.unique(idx)), m)
    op = reduced.build_operator(m, phi, q_ref, d, samp)
    a = reduced.encode(op, u0)
    y_corr = u0
    tm = {}

    def timed(name, fn, *args):
        t = time.perf_counter()
        out = fn(*args)
        tm[name] = time.perf_counter() - t
        return out

    t0 = time.perf_counter()
    out = timed("lspg_step", reduced.lspg_step, op, m, a, case.dt, 1e-8, 10)       # driver.py:338
    q_tilde = timed("decode", reduced.decode, op, out.a)                            # :343
    res = timed("coarse_step", physics.coarse_step, m, y_corr, case.z, case.dt)     # :354
    y_hat = d * (res.x - q_ref)                                                     # :359
    phi2, sig2, _ = timed("isvd_update", subspace.isvd_update, phi, sigma, y_hat,
                          case.lam, r)                                              # :365
    timed("residual_norm", lambda: float(np.linalg.norm(y_hat - phi @ (phi.T @ y_hat))))  # :366
    samp2 = timed("qdeim_sample", online._sampling, ocfg, phi2, res.x)              # :370
    op2 = timed("build_operator", reduced.build_operator, m, phi2, q_ref, d, samp2)  # :373
    timed("encode", reduced.encode, op2, q_tilde)                                   # :376
    step = time.perf_counter() - t0
    n_online = case.n_t - case.w_init
    start = tm["coarse_step"] + tm["qdeim_sample"] + tm["build_operator"] + tm["encode"]
    per_step = step + start / n_online
    return per_step, {"components_s": {k: round(v, 3) for k, v in tm.items()},
                      "step_s": round(step, 3), "gn_iterations": int(out.iterations),
                      "sample": f"one online step of the oracle loop at N={n} (the benchmarked "
                                f"grid), every component once ({step:.1f} s); start (= coarse "
                                f"step + QDEIM + operator + encode) amortised over {n_online} "
                                f"online steps; synthetic offline stand-ins of the real shapes "
                                f"(bench.cpu_step_full_grid)"}


def cpu_baseline_rom(case, steps=100):
    """The host-core baseline at the benchmarked configuration: the oracle
    loop at the case's own grid (cfg 0 / 1), or one full-grid step by
    components (cfg 3).  Configuration 4 has no reference model; its port
    runs on a 2^12-cell sample scaled in N (same_config false)."""
    if case.model == "reacting":
        n_sample = 1 << 12
        small, ocfg = _oracle_loop_config(case, n_sample, steps)
        from oracle import online
        training = online.training_states(ocfg, small.initial_state())
        q_ref, d, phi0, sigma0 = online.offline(ocfg, training)
        t0 = time.perf_counter()
        online.run_online(ocfg, training, q_ref, d, phi0, sigma0, keep_stride=10 ** 9, n_steps=steps)
        per = (time.perf_counter() - t0) / steps * (case.n_elem / n_sample)
        return {"value": round(1.0 / per, 6), "unit": "online steps/s", "cores": cpu_cores(),
                "kind": "port", "same_config": False,
                "sample": f"oracle loop of the builder-defined reacting model at N={n_sample}, "
                          f"{steps} steps incl. start, scaled x{case.n_elem // n_sample} in N "
                          f"(no reference model exists, SPEC.md:8)"}
    if case.n_elem <= (1 << 16):
        per, det = cpu_loop_rom(case, steps)
    else:
        per, det = cpu_step_full_grid(case)
    out = {"value": round(1.0 / per, 6), "unit": "online steps/s", "cores": cpu_cores(),
           "kind": "port", "same_config": True}
    out.update(det)
    return out


def reference_rom(args, rank, world):
    """--impl reference: the reference's algorithm (the oracle port; the
    reference package itself cannot run past N ~ 4000: dense N^2 Newton) on
    the host cores at the benchmarked configuration.  For configuration 3
    one full-grid online step (~2 min) is the bounded sample, so `steps`
    reports the steps actually timed."""
    if rank != 0:
        return None
    case = rom_case(args.config, args.n)
    steps = 100 if case.n_elem <= (1 << 16) else 1
    base = cpu_baseline_rom(case, steps=steps)
    value = base["value"]
    return {
        "metric": ROM_METRIC, "impl": "reference", "value": value, "unit": "online steps/s",
        "n_gpus": world, "steps": steps, "warmup": 0,
        "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": round(1e3 / value, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": case.name, "n_elem": case.n_elem, "r": case.r, "n_s": case.n_s,
                   "z": case.z},
        "cpu_baseline": base,
        "e2e": {"value": value, "unit": "online steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


# --------------------------------------------------------------------------- main

# --------------------------------------------------------------------------- cfg4

CFG4_METRIC = "reacting Euler residual Gcell/s (cfg4: 2^20 cells x 13 vars)"


def bench_cfg4(args, rank, world):
    """Configuration-4 residual alone (`--config cfg4-residual`; SURVEY §8a
    row a3, §8d: 208 B/cell): a step = one residual evaluation over the grid.
    The full configuration-4 adaptive loop is `--config cfg4` (bench_rom).
    The reference has no such model, so there is no reference arm
    (cpu_baseline: the numpy oracle that defines the model, timed on a
    bounded sample)."""
    import torch
    import paper_2605_28684_b200 as P
    from paper_2605_28684_b200 import _lib
    n = args.n or (1 << 20)
    m = P.ReactingEulerProblem(n)
    q = torch.from_numpy(m.initial_state()).cuda()
    out = torch.empty_like(q)
    ctx = _lib.Context.get()
    mabi = m.abi()
    import ctypes as C
    call = lambda: ctx.call("adrom_rhs", C.byref(mabi), _lib.ptr(q), _lib.ptr(out))  # noqa: E731
    for _ in range(max(args.warmup, 3)):
        call()
    torch.cuda.synchronize()
    barrier(world)
    K = max(args.steps, 20)
    l0 = ctx.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        ev0.record()
        for _ in range(K):
            call()
        ev1.record()
        torch.cuda.synchronize()
    ms = max_over_ranks(ev0.elapsed_time(ev1), world) / K
    gcells = world * n / (ms * 1e-3) / 1e9
    line = {
        "metric": CFG4_METRIC, "value": round(gcells, 2), "unit": "Gcell/s", "n_gpus": world,
        "steps": K, "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded mechanism and pulse IC, DESIGN.md §9)",
        "config": {"workload": "cfg4-reacting-residual-2^20", "n_elem": n, "n_var": 13,
                   "l2": "inputs larger than L2 (%.0f MB state)" % (8 * 13 * n / 1e6),
                   "parallelism": f"replicas{world}"},
        "roofline": roofline(208.0 * n, ms),
        "gpu_launches": ctx.launches() - l0,
        "clocks": clk.summary(),
    }
    line["roofline"]["kernel"] = "reacting_rhs_kernel (208 B/cell)"
    # one backward-Euler step on the same grid (a4 for configuration 4)
    dt4 = 2e-5
    P.implicit_step(m, q, dt4)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = P.implicit_step(m, q, dt4)
    e1.record()
    torch.cuda.synchronize()
    line["implicit_step"] = {"ms": round(e0.elapsed_time(e1), 3), "dt": dt4,
                             "iterations": int(res.iterations), "converged": bool(res.converged)}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import reacting as R
        ns = 1 << 16
        qh = R.initial_state(ns)
        t0 = time.perf_counter()
        reps = 0
        while time.perf_counter() - t0 < 5.0:
            R.rhs(qh, ns, 1.0 / ns, 1.4, R.mechanism())
            reps += 1
        dt = (time.perf_counter() - t0) / reps
        line["cpu_baseline"] = {"value": round(ns / dt / 1e9, 5), "unit": "Gcell/s", "cores": 1,
                                "kind": "port",
                                "sample": f"oracle/reacting.rhs (numpy) at 2^16 cells, {reps} reps"}
    return line


def reference_cfg4(args, rank, world):
    return {"impl": "reference",
            "unavailable": "the reference has no reacting model (SPEC.md:8); see cpu_baseline"}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3", choices=["cfg0", "cfg1", "cfg2", "cfg3", "cfg4",
                                                         "cfg4-residual"])
    ap.add_argument("--n-elem", dest="n", type=int, default=0, help="override grid size (testing)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", dest="e2e_steps", type=int, default=0,
                    help="online steps of the e2e run (0: the default horizon)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        print("warning: the contract asks for >= 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        fn = {"cfg2": reference_cfg2, "cfg0": reference_rom, "cfg1": reference_rom,
              "cfg3": reference_rom, "cfg4": reference_rom,
              "cfg4-residual": reference_cfg4}.get(args.config)
        line = fn(args, rank, world) if fn else None
        if rank == 0:
            print(json.dumps(line if line else {"impl": "reference",
                                                "unavailable": f"{args.config} not wired yet"}))
        return 0
    rank, world, _ = dist_setup()
    fn = {"cfg2": bench_cfg2, "cfg0": bench_rom, "cfg1": bench_rom, "cfg3": bench_rom,
          "cfg4": bench_rom, "cfg4-residual": bench_cfg4}[args.config]
    line = fn(args, rank, world)
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
