"""Artifact writers (paper_2605_28684_b200.io) against the bytes the
reference's own writers produce (tests/golden/io_artifacts.npz, made by
tests/golden/make_golden.py io_artifacts from /root/reference io.py:65-205)."""

import json

import numpy as np

import paper_2605_28684_b200 as P
from paper_2605_28684_b200 import io as pio


def _result(g):
    cfg = P.ExperimentConfig(model="sod", n_elem=16, dt=1e-3, n_t=24, w_init=8, r=4, n_s=6, z=4,
                             sampling="fgs", n_extra=2, rule=P.UpdateRule("isvd", lam=0.25),
                             save_stride=5, label="golden-io")
    return P.RunResult(config=cfg, kind="adaptive", trajectory=g["traj"], wall_seconds=0.125,
                       var_names=("rho", "v", "p"), newton_failures=[11, 17],
                       error_steps=np.arange(9, 25), errors=g["errors"],
                       event_log=[{"event": 1, "step": 12, "coarse_converged": True,
                                   "coarse_iterations": 3, "residual_norm": 0.5}],
                       signal_steps=g["sig_steps"], signal_errors=g["sig_err"])


def test_artifacts_byte_identical(golden, tmp_path):
    g = golden("io_artifacts")
    res = _result(g)
    run_dir = tmp_path / "run-golden"
    run_dir.mkdir()
    writers = {"error_history.csv": pio.write_error_history,
               "signal_errors.csv": pio.write_signal_errors,
               "profiles.csv": pio.write_profiles, "snapshots.csv": pio.write_snapshots}
    for name, fn in writers.items():
        fn(run_dir / name, res)
        assert (run_dir / name).read_text() == str(g["file_" + name]), name
    pio.write_manifest(run_dir, res, list(writers), fom_wall=1.5)
    assert (run_dir / "manifest.json").read_text() == str(g["file_manifest.json"])


def test_config_roundtrip_and_cache_key(golden):
    g = golden("io_artifacts")
    cfg = _result(g).config
    d = pio.config_to_dict(cfg)
    assert json.dumps(d) == str(g["config_dict"])
    assert pio.config_from_dict(d) == cfg
    assert pio.fom_cache_key(cfg) == str(g["cache_key"])


def test_load_error_history_roundtrip(golden, tmp_path):
    g = golden("io_artifacts")
    res = _result(g)
    pio.write_error_history(tmp_path / "e.csv", res)
    header, data = pio.load_error_history(tmp_path / "e.csv")
    assert header == ["step", "time", "rho_rel_err", "v_rel_err", "p_rel_err"]
    assert np.array_equal(data[:, 2:], g["errors"]) and np.array_equal(data[:, 0], np.arange(9, 25))
