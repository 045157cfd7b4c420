"""ctypes binding of ``lib/libadrom_b200.so`` (C-ABI: ``include/adrom_b200.h``).

The product path has no CPU fallback: if the shared library is missing or
no CUDA device is visible, every entry point raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from .errors import DenseError, RomStepError

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "lib" / "libadrom_b200.so"

OK, ERR_NONFINITE, ERR_SINGULAR, ERR_ROMSTEP, ERR_ARG, ERR_CUDA, ERR_NOCONV, ERR_DENSE = range(8)
BURGERS, SOD, REACTING = 1, 2, 3

_p = C.c_void_p
_i32, _i64, _f64 = C.c_int32, C.c_int64, C.c_double


class Model(C.Structure):
    """``adrom_model`` (include/adrom_b200.h)."""

    _fields_ = [("kind", _i32), ("n_var", _i32), ("n_elem", _i64),
                ("dx", _f64), ("nu", _f64), ("gamma", _f64), ("mech", _p)]


class NewtonInfo(C.Structure):
    _fields_ = [("converged", _i32), ("iterations", _i32), ("residual_norm", _f64)]


class IsvdInfo(C.Structure):
    _fields_ = [("qnorm", _f64), ("ynorm", _f64), ("proj_resid", _f64),
                ("degenerate", _i32), ("reorthogonalised", _i32), ("sweeps", _i32),
                ("core_path", _i32)]


class RomOp(C.Structure):
    """``adrom_rom_op`` — device buffers of a reduced operator."""

    _fields_ = [("r", _i32), ("n_var", _i32), ("ns_cap", _i32), ("nc_cap", _i32),
                ("ncell_cap", _i32), ("pad", _i32),
                ("idx", _p), ("closure", _p), ("gather", _p), ("out_cell", _p),
                ("out_var", _p), ("sample_pos", _p), ("sizes", _p),
                ("pinv", _p), ("d_s", _p), ("q_ref_c", _p), ("dinv_phi_c", _p), ("phi_s", _p)]


class RomStepInfo(C.Structure):
    _fields_ = [("converged", _i32), ("iterations", _i32), ("residual_norm", _f64)]


class SessionConfig(C.Structure):
    """``adrom_session_config``."""

    _fields_ = [("model", Model), ("r", _i32), ("n_s", _i32), ("n_extra", _i32), ("z", _i32),
                ("projection", _i32), ("sampling", _i32), ("feature", _i32), ("adaptive", _i32),
                ("newton_max_iter", _i32), ("pad", _i32), ("w_init", _i64), ("n_t", _i64),
                ("dt", _f64), ("lam", _f64), ("newton_tol", _f64)]


class EventRecord(C.Structure):
    _fields_ = [("step", _i64), ("coarse_converged", _i32), ("coarse_iterations", _i32),
                ("residual_norm", _f64), ("error", _i32), ("pad", _i32)]


# name -> (restype, argtypes)
SIGNATURES = {
    "adrom_abi_version": (_i32, []),
    "adrom_ctx_create": (_i32, [C.POINTER(_p), _p]),
    "adrom_ctx_set_stream": (_i32, [_p, _p]),
    "adrom_ctx_destroy": (None, [_p]),
    "adrom_ctx_last_error": (C.c_char_p, [_p]),
    "adrom_ctx_synchronize": (_i32, [_p]),
    "adrom_ctx_launch_count": (_i64, [_p]),
    "adrom_prof_enable": (_i32, [_p, _i32]),
    "adrom_prof_read": (_i32, [_p, C.POINTER(_f64), C.POINTER(_i32)]),
    "adrom_rhs": (_i32, [_p, C.POINTER(Model), _p, _p]),
    "adrom_rhs_at_cells": (_i32, [_p, C.POINTER(Model), _p, _i64, _p]),
    "adrom_plan_evaluate": (_i32, [_p, C.POINTER(Model), _p, _i64, _p, _p, _i64, _p, _p, _p,
                                   _i64, _i32, _p]),
    "adrom_fd_jacobian_blocks": (_i32, [_p, C.POINTER(Model), _p, _p]),
    "adrom_implicit_step": (_i32, [_p, C.POINTER(Model), _p, _f64, _f64, _i32, _p,
                                   C.POINTER(NewtonInfo)]),
    "adrom_project": (_i32, [_p, _p, _p, _i64, _i32, _p]),
    "adrom_encode": (_i32, [_p, _p, _p, _p, _p, _i64, _i32, _p]),
    "adrom_decode": (_i32, [_p, _p, _p, _p, _p, _i64, _i32, _p]),
    "adrom_isvd_update": (_i32, [_p, _p, _p, _p, _i64, _i32, _i32, _f64, _p, _p, _p,
                                 C.POINTER(IsvdInfo)]),
    "adrom_gram": (_i32, [_p, _p, _i64, _i32, _p]),
    "adrom_isvd_stream_create": (_i32, [_p, _i64, _i32, C.POINTER(_p)]),
    "adrom_isvd_stream_destroy": (None, [_p]),
    "adrom_isvd_stream_load": (_i32, [_p, _p, _p]),
    "adrom_isvd_stream_update": (_i32, [_p, _p, _f64, C.POINTER(IsvdInfo)]),
    "adrom_isvd_stream_read": (_i32, [_p, _p, _p]),
    "adrom_small_svd": (_i32, [_p, _p, _i32, _i32, _p, _p, _p]),
    "adrom_ts_tn": (_i32, [_p, _i64, _i32, _i32, _p, _i64, _i32, _p, _i64, _p]),
    "adrom_ts_apply": (_i32, [_p, _i64, _i32, _i32, _p, _i64, _p, _p, _i64, _i32]),
    "adrom_fit_scaling": (_i32, [_p, _p, _i32, _i64, _i32, _p, _p]),
    "adrom_pod_window": (_i32, [_p, _p, _i32, _i64, _i32, _p, _p, _i32, _p, _p, _p,
                                C.POINTER(_i32)]),
    "adrom_pod": (_i32, [_p, _p, _i64, _i32, _i32, _p, _p, _p, C.POINTER(_i32)]),
    "adrom_orth": (_i32, [_p, _p, _i64, _i32, _p]),
    "adrom_least_squares": (_i32, [_p, _p, _i64, _i32, _p, _i32, _p]),
    "adrom_rusanov_flux": (_i32, [_p, _p, _p, _i64, _f64, _p]),
    "adrom_lu_solve": (_i32, [_p, _p, _i64, _p]),
    "adrom_qdeim": (_i32, [_p, _p, _i64, _i32, _i32, _p]),
    "adrom_fgs": (_i32, [_p, C.POINTER(Model), _p, _i32, _p, _i32, _i32, _i32, _p]),
    "adrom_deim_operator": (_i32, [_p, _p, _i64, _i32, _p, _i32, _p]),
    "adrom_rom_operator_build": (_i32, [_p, C.POINTER(Model), _p, _i64, _p, _p, _p, _i32,
                                        C.POINTER(RomOp)]),
    "adrom_rom_step": (_i32, [_p, C.POINTER(Model), C.POINTER(RomOp), _i32, _p, _f64, _f64,
                              _i32, _p, C.POINTER(RomStepInfo)]),
    "adrom_session_create": (_i32, [_p, C.POINTER(SessionConfig), C.POINTER(_p)]),
    "adrom_session_destroy": (None, [_p]),
    "adrom_session_load": (_i32, [_p, _p, _p, _p, _p, _p]),
    "adrom_session_start": (_i32, [_p]),
    "adrom_session_advance": (_i32, [_p, _i64, _i64, _p, _p, C.POINTER(_i64)]),
    "adrom_session_finish": (_i32, [_p]),
    "adrom_session_read": (_i32, [_p, _p, _i64, _p, _i64, C.POINTER(_i64), C.POINTER(_i64),
                                  _p, _p, _p, _p]),
    "adrom_session_sampling": (_i32, [_p, _p]),
    "adrom_session_set_host_ring": (_i32, [_p, _i64]),
    "adrom_session_signal": (_i32, [_p, _p]),
    "adrom_state_errors": (_i32, [_p, C.POINTER(Model), _p, _p, _p]),
}

PROBES = ["isvd_rotate", "isvd_project", "isvd_resid", "isvd_core", "fom_residual",
          "fom_jacobian", "fom_solve", "qdeim_round", "rom_step", "decode", "operator", "encode",
          "isvd_small", "isvd_reanchor"]

_lib = None
_lock = threading.Lock()


def load(path: str | os.PathLike | None = None) -> C.CDLL:
    """Load the C-ABI library (fail loudly if it is absent)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise RuntimeError(
                f"{p} is missing: build it with `python -m paper_2605_28684_b200._build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def exported_symbols(path=None) -> set[str]:
    """Names from SIGNATURES that the library exports (no GPU needed)."""
    lib = C.CDLL(str(Path(path) if path else LIB_PATH))
    return {n for n in SIGNATURES if hasattr(lib, n)}


class Context:
    """One ``adrom_ctx`` per (device, thread); rebinds to torch's current stream."""

    _tls = threading.local()

    def __init__(self):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2605_28684_b200 needs a CUDA device (no CPU fallback)")
        self.lib = load()
        handle = _p()
        st = self.lib.adrom_ctx_create(C.byref(handle), _p(torch.cuda.current_stream().cuda_stream))
        if st != OK:
            raise RuntimeError(f"adrom_ctx_create failed with status {st}")
        self.handle = handle
        self._stream = None

    @classmethod
    def get(cls) -> "Context":
        import torch
        dev = torch.cuda.current_device()
        table = getattr(cls._tls, "table", None)
        if table is None:
            table = cls._tls.table = {}
        ctx = table.get(dev)
        if ctx is None:
            ctx = table[dev] = cls()
        ctx.bind()
        return ctx

    def bind(self):
        import torch
        s = torch.cuda.current_stream().cuda_stream
        if s != self._stream:
            self.lib.adrom_ctx_set_stream(self.handle, _p(s))
            self._stream = s

    def error(self) -> str:
        msg = self.lib.adrom_ctx_last_error(self.handle)
        return msg.decode() if msg else ""

    def check(self, status: int, what: str = ""):
        if status == OK:
            return
        msg = self.error() or what
        if status in (ERR_NONFINITE, ERR_SINGULAR, ERR_NOCONV, ERR_DENSE):
            raise DenseError(msg)
        if status == ERR_ROMSTEP:
            raise RomStepError(msg)
        if status == ERR_ARG:
            raise ValueError(msg)
        raise RuntimeError(f"CUDA failure in {what}: {msg}")

    def call(self, name: str, *args):
        self.check(getattr(self.lib, name)(self.handle, *args), name)

    def scall(self, name: str, session, *args):
        """Call a session entry point (first argument is the session handle)."""
        self.check(getattr(self.lib, name)(session, *args), name)

    def sync(self):
        self.call("adrom_ctx_synchronize")

    def launches(self) -> int:
        return int(self.lib.adrom_ctx_launch_count(self.handle))

    def prof_enable(self, on: bool = True):
        self.call("adrom_prof_enable", _i32(1 if on else 0))

    def prof_read(self) -> dict:
        ms = (_f64 * 16)()
        cnt = (_i32 * 16)()
        self.call("adrom_prof_read", ms, cnt)
        return {PROBES[i]: (ms[i], cnt[i]) for i in range(len(PROBES)) if cnt[i]}


def ptr(t) -> _p:
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return _p(0)
    return _p(t.data_ptr())


def model_struct(kind: int, n_var: int, n_elem: int, dx: float, nu: float, gamma: float,
                 mech=None) -> Model:
    return Model(kind, n_var, n_elem, dx, nu, gamma, ptr(mech))


__all__ = ["Context", "load", "ptr", "Model", "NewtonInfo", "IsvdInfo", "SIGNATURES",
           "exported_symbols", "np"]
