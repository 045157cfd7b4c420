"""FP64 tensor-core GEMMs (csrc/dgemm.cu) vs numpy, and the DMMA rotation at
r = 128 vs the CUDA-core rotation.  The large-sample reduced operator of
configuration 4 (DEIM pseudo-inverse, sampling.py:162-175; Gauss-Newton
contraction, projection.py:176/187) runs on these kernels instead of cuBLAS."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rel(got, want):
    return np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300)


@pytest.mark.parametrize("k,m,n,akm", [(408_954, 128, 129, True), (408_954, 128, 128, False),
                                       (1000, 13, 37, False), (1001, 100, 136, True),
                                       (5, 128, 136, False), (33, 1, 1, True)])
def test_ts_tn_vs_numpy(k, m, n, akm):
    from paper_2605_28684_b200 import _dev
    from paper_2605_28684_b200.dense import ts_tn
    rng = np.random.default_rng(k + m + n)
    a = rng.standard_normal((m, k) if akm else (k, m))
    b = rng.standard_normal((k, n))
    got = _dev.host(ts_tn(a, b, a_kmajor=akm))
    want = (a @ b) if akm else (a.T @ b)
    # error of a length-K fp64 dot product: ~ sqrt(K) eps |a||b| per entry
    scale = np.sqrt(np.outer((a * a).sum(1) if akm else (a * a).sum(0), (b * b).sum(0)))
    assert np.all(np.abs(got - want) <= 1e-13 * max(1.0, np.sqrt(k) / 8) * scale + 1e-300)
    again = _dev.host(ts_tn(a, b, a_kmajor=akm))
    assert np.array_equal(got, again), "split-K sum is not deterministic"


def test_ts_tn_empty_k():
    from paper_2605_28684_b200 import _dev
    from paper_2605_28684_b200.dense import ts_tn
    got = _dev.host(ts_tn(np.zeros((0, 7)), np.zeros((0, 9))))
    assert got.shape == (7, 9) and not got.any()


@pytest.mark.parametrize("k,m,n,kmaj", [(408_954, 128, 128, True), (408_954, 128, 128, False),
                                        (1001, 7, 129, False), (31, 128, 136, True)])
def test_ts_apply_vs_numpy(k, m, n, kmaj):
    from paper_2605_28684_b200 import _dev
    from paper_2605_28684_b200.dense import ts_apply
    rng = np.random.default_rng(7 * k + m)
    a = rng.standard_normal((k, m))
    mm = rng.standard_normal((m, n))
    got = _dev.host(ts_apply(a, mm, out_kmajor=kmaj))
    want = a @ mm
    if kmaj:
        got = got.T
    scale = np.sqrt(np.outer((a * a).sum(1), (mm * mm).sum(0)))
    assert np.all(np.abs(got - want) <= 1e-14 * m * scale + 1e-300)


def test_rotation_r128_tensor_core_matches_cuda_core(monkeypatch):
    """isvd_update at r = 128: the DMMA rotation (rot_tc_kernel<128>) and the
    CUDA-core one (ADROM_NO_TC_ROT) give the same basis to rounding."""
    from paper_2605_28684_b200 import ReducedBasis, _dev, isvd_update
    from oracle import subspace
    rng = np.random.default_rng(128)
    n, r = 1 << 16, 128
    phi = np.linalg.qr(rng.standard_normal((n, r)))[0]
    sig = np.sort(rng.uniform(0.5, 3.0, r))[::-1]
    y = phi @ rng.standard_normal(r) + 0.3 * rng.standard_normal(n)
    tc = isvd_update(ReducedBasis(phi, sig), y, 0.8, r)
    monkeypatch.setenv("ADROM_NO_TC_ROT", "1")
    cc = isvd_update(ReducedBasis(phi, sig), y, 0.8, r)
    assert np.allclose(tc.sigma, cc.sigma, rtol=1e-13)
    assert np.max(np.abs(np.asarray(tc.phi) - np.asarray(cc.phi))) < 1e-13
    ref_phi, ref_sig, _ = subspace.isvd_update(phi, sig, y, 0.8, r)
    assert np.allclose(tc.sigma, ref_sig, rtol=1e-10)
    assert subspace.max_angle(ref_phi, np.asarray(tc.phi)) < 1e-9
