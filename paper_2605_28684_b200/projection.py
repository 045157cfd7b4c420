"""Reduced operators and reduced steps with the reference signatures
(``adrom/projection.py``), backed by device buffers.

``RomOperator`` owns the ``adrom_rom_op`` buffers (closure, gather plan,
DEIM pseudo-inverse, closure-restricted basis, ...) built on the device by
``adrom_rom_operator_build``; ``lspg_step`` / ``galerkin_step`` run the whole
nonlinear iteration in one thread block (``adrom_rom_step``).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _dev
from ._lib import Context, RomOp, RomStepInfo, ptr
from .errors import RomStepError
from .sampling import SamplingPlan, SamplingSet

__all__ = ["ReducedState", "RomOperator", "RomStepResult", "RomStepError", "build_rom_operator",
           "encode", "decode", "galerkin_step", "lspg_step", "rom_step", "lspg_objective"]


@dataclass(frozen=True)
class ReducedState:
    """projection.py:41-46."""

    a: object
    n: int = 0


@dataclass(frozen=True)
class RomStepResult:
    """projection.py:49-54."""

    state: ReducedState
    converged: bool
    iterations: int
    residual_norm: float


class RomOperator:
    """projection.py:57-87 on the device."""

    def __init__(self, basis, scaling, sampling: SamplingSet, model, kind: str):
        if kind not in ("galerkin", "lspg"):
            raise ValueError(f"unknown projection kind {kind!r}")
        t = _dev.torch()
        self.basis = basis
        self.scaling = scaling
        self.sampling = sampling
        self.kind = kind
        self.model = model
        # the reference requires the closure to cover the stencil (fom.py:140-144)
        self.plan = SamplingPlan(model, sampling)
        phi = _dev.dev(basis.phi)
        n, r = phi.shape
        nv = model.n_var
        n_s = sampling.n_samples
        nc = 3 * n_s * nv
        i64 = t.int64
        self._buf = dict(
            idx=_dev.dev_i64(sampling.indices), closure=_dev.empty(nc, dtype=i64),
            gather=_dev.empty(n_s * 3 * nv, dtype=i64), out_cell=_dev.empty(n_s, dtype=i64),
            out_var=_dev.empty(n_s, dtype=i64), sample_pos=_dev.empty(n_s, dtype=i64),
            sizes=_dev.zeros(4, dtype=t.int32), pinv=_dev.empty(r * n_s), d_s=_dev.empty(n_s),
            q_ref_c=_dev.empty(nc), dinv_phi_c=_dev.empty(nc * r), phi_s=_dev.empty(n_s * r))
        b = self._buf
        self.op = RomOp(r, nv, n_s, nc, n_s, 0, *(b[k].data_ptr() for k in (
            "idx", "closure", "gather", "out_cell", "out_var", "sample_pos", "sizes", "pinv",
            "d_s", "q_ref_c", "dinv_phi_c", "phi_s")))
        q_ref = _dev.dev(scaling.q_ref)
        d = _dev.dev(scaling.row_scale)
        self._keep = (phi, q_ref, d)
        m = model.abi()
        Context.get().call("adrom_rom_operator_build", C.byref(m), ptr(phi), C.c_int64(n), ptr(q_ref),
                           ptr(d), None, C.c_int32(n_s), C.byref(self.op))
        sizes = _dev.host(b["sizes"])
        self._n_s, self._n_c = int(sizes[0]), int(sizes[1])
        self._r = r

    @property
    def rank(self) -> int:
        return self._r

    # host views with the reference's attribute names -----------------------
    @property
    def deim_pinv(self):
        return _dev.host(self._buf["pinv"][: self._r * self._n_s].reshape(self._r, self._n_s))

    @property
    def d_sampled(self):
        return _dev.host(self._buf["d_s"][: self._n_s])

    @property
    def phi_sampled(self):
        return _dev.host(self._buf["phi_s"][: self._n_s * self._r].reshape(self._n_s, self._r))

    # The device kernels gather through the stencil closure of the sampled
    # rows (sampling.py:178-189).  A caller-supplied closure that is a strict
    # superset of it (projection.py:73-79 takes sampling.closure verbatim)
    # changes nothing the operator computes, only these arrays' extent, so
    # the views are then formed from sampling.closure like the reference's.
    def _user_closure(self):
        clo = np.asarray(self.sampling.closure, dtype=np.int64)
        dev_clo = _dev.host(self._buf["closure"][: self._n_c])
        return None if np.array_equal(clo, dev_clo) else clo

    @property
    def closure(self):
        clo = self._user_closure()
        return clo if clo is not None else _dev.host(self._buf["closure"][: self._n_c])

    @property
    def q_ref_closure(self):
        clo = self._user_closure()
        if clo is not None:
            return np.asarray(_dev.host(self.scaling.q_ref))[clo]
        return _dev.host(self._buf["q_ref_c"][: self._n_c])

    @property
    def dinv_phi_closure(self):
        clo = self._user_closure()
        if clo is not None:
            d = np.asarray(_dev.host(self.scaling.row_scale))
            return np.asarray(_dev.host(self.basis.phi))[clo, :] / d[clo][:, None]
        return _dev.host(self._buf["dinv_phi_c"][: self._n_c * self._r].reshape(self._n_c, self._r))

    @property
    def sample_pos(self):
        clo = self._user_closure()
        if clo is not None:
            return np.searchsorted(clo, np.asarray(self.sampling.indices))
        return _dev.host(self._buf["sample_pos"][: self._n_s])

    def decode_closure(self, a):
        """projection.py:86-87 (on the device closure, or on a caller-supplied
        superset closure)."""
        clo = self._user_closure()
        if clo is not None:
            t = _dev.torch()
            ci = t.from_numpy(clo).cuda()
            d = _dev.dev(self.scaling.row_scale)[ci]
            dphi = _dev.dev(self.basis.phi)[ci] / d[:, None]
            from .dense import ts_apply
            qc = _dev.dev(self.scaling.q_ref)[ci] + ts_apply(dphi.contiguous(), _dev.dev(a)[:, None]).reshape(-1)
            return _dev.like(qc, a)
        qc = self._buf["q_ref_c"][: self._n_c] + \
            self._buf["dinv_phi_c"][: self._n_c * self._r].reshape(self._n_c, self._r) @ _dev.dev(a)
        return _dev.like(qc, a)


def build_rom_operator(basis, scaling, sampling, model, kind) -> RomOperator:
    """projection.py:90-93."""
    return RomOperator(basis, scaling, sampling, model, kind)


def encode(q, op: RomOperator, n: int = 0) -> ReducedState:
    """projection.py:96-99 — a = phi^T D (q - q_ref) (``adrom_encode``)."""
    phi = _dev.dev(op.basis.phi)
    nn, r = phi.shape
    a = _dev.empty(r)
    q_ref, d = _dev.dev(op.scaling.q_ref), _dev.dev(op.scaling.row_scale)
    qd = _dev.dev(q)
    Context.get().call("adrom_encode", ptr(phi), ptr(q_ref), ptr(d), ptr(qd),
                       C.c_int64(nn), C.c_int32(r), ptr(a))
    return ReducedState(a=_dev.like(a, q), n=n)


def decode(state: ReducedState, op: RomOperator):
    """projection.py:102-104 — q_ref + (phi a) / d (``adrom_decode``)."""
    phi = _dev.dev(op.basis.phi)
    nn, r = phi.shape
    out = _dev.empty(nn)
    q_ref, d = _dev.dev(op.scaling.q_ref), _dev.dev(op.scaling.row_scale)
    ad = _dev.dev(state.a)
    Context.get().call("adrom_decode", ptr(phi), ptr(q_ref), ptr(d), ptr(ad),
                       C.c_int64(nn), C.c_int32(r), ptr(out))
    return _dev.like(out, state.a)


def _step(op: RomOperator, model, state: ReducedState, dt, tol, max_iter, kind) -> RomStepResult:
    a_prev = _dev.dev(state.a)
    a_out = _dev.empty(op.rank)
    info = RomStepInfo()
    m = model.abi()
    Context.get().call("adrom_rom_step", C.byref(m), C.byref(op.op), C.c_int32(kind), ptr(a_prev),
                       C.c_double(dt), C.c_double(tol), C.c_int32(max_iter), ptr(a_out),
                       C.byref(info))
    return RomStepResult(state=ReducedState(a=_dev.like(a_out, state.a), n=state.n + 1),
                         converged=bool(info.converged), iterations=int(info.iterations),
                         residual_norm=float(info.residual_norm))


def lspg_step(op, model, state, dt, tol=1e-8, max_iter=10) -> RomStepResult:
    """projection.py:158-204."""
    return _step(op, model, state, dt, tol, max_iter, 0)


def galerkin_step(op, model, state, dt, tol=1e-8, max_iter=10) -> RomStepResult:
    """projection.py:111-147."""
    return _step(op, model, state, dt, tol, max_iter, 1)


def rom_step(op, model, state, dt, tol=1e-8, max_iter=10) -> RomStepResult:
    """projection.py:217-221."""
    if op.kind == "galerkin":
        return galerkin_step(op, model, state, dt, tol=tol, max_iter=max_iter)
    return lspg_step(op, model, state, dt, tol=tol, max_iter=max_iter)


def lspg_objective(op: RomOperator, state_prev: ReducedState, a, dt: float) -> float:
    """projection.py:207-214 (diagnostic)."""
    pos = op._buf["sample_pos"][: op._n_s]
    prev_s = _dev.dev(op.decode_closure(_dev.dev(state_prev.a)))[pos]
    qc = _dev.dev(op.decode_closure(_dev.dev(a)))
    fs = _evaluate_on_device_closure(op, qc)
    res = op._buf["d_s"][: op._n_s] * (qc[pos] - prev_s - dt * fs)
    rho = op._buf["pinv"][: op.rank * op._n_s].reshape(op.rank, op._n_s) @ res
    return float((rho @ rho).item())


def _evaluate_on_device_closure(op: RomOperator, qc):
    """Sampled rhs from values on the device closure (sizes[1] rows)."""
    from ._lib import ptr as _ptr
    b = op._buf
    m = op.model.abi()
    out = _dev.empty(op._n_s)
    Context.get().call("adrom_plan_evaluate", C.byref(m), _ptr(b["gather"]),
                       C.c_int64(op._n_s), _ptr(b["out_cell"]), _ptr(b["out_var"]),
                       C.c_int64(op._n_s), _ptr(qc), None, None, C.c_int64(0), C.c_int32(0),
                       _ptr(out))
    return out
