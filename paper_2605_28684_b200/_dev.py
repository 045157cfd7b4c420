"""Host <-> device plumbing for the reference-shaped API.

Functions of the public API accept numpy arrays (host, like the reference)
or torch CUDA tensors (device-resident fast path) and return the same kind
they were given.  torch supplies device memory and streams only; all
arithmetic happens in the C-ABI library.
"""

from __future__ import annotations

import numpy as np


def torch():
    import torch as _t
    return _t


def is_device(x) -> bool:
    t = torch()
    return isinstance(x, t.Tensor) and x.is_cuda


def dev(x, dtype=None):
    """Contiguous CUDA tensor (float64 unless dtype given) holding x."""
    t = torch()
    dtype = dtype or t.float64
    if isinstance(x, t.Tensor):
        y = x.to(device="cuda", dtype=dtype)
        return y.contiguous()
    arr = np.ascontiguousarray(np.asarray(x))
    return t.from_numpy(arr).to(device="cuda", dtype=dtype).contiguous()


def dev_i64(x):
    return dev(x, dtype=torch().int64)


def empty(*shape, dtype=None):
    t = torch()
    return t.empty(*shape, dtype=dtype or t.float64, device="cuda")


def zeros(*shape, dtype=None):
    t = torch()
    return t.zeros(*shape, dtype=dtype or t.float64, device="cuda")


def host(x) -> np.ndarray:
    t = torch()
    if isinstance(x, t.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def like(result, template):
    """Return ``result`` (a CUDA tensor) as the kind ``template`` is."""
    return result if is_device(template) else host(result)
