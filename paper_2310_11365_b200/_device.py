"""Device plumbing: torch is used for device memory and streams only."""

from __future__ import annotations

import torch

from ._lib import MmprError


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise MmprError("no CUDA device: the mM-Parareal hot path runs only on the GPU (no CPU fallback)")


def device() -> torch.device:
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def empty(shape, dtype=torch.float64):
    return torch.empty(shape, dtype=dtype, device=device())


def zeros(shape, dtype=torch.float64):
    return torch.zeros(shape, dtype=dtype, device=device())


def as_device_f64(values) -> torch.Tensor:
    """Contiguous float64 device copy of array-like ``values`` (1-D)."""
    if isinstance(values, torch.Tensor):
        t = values.detach()
        if t.device.type != "cuda" or t.dtype != torch.float64:
            t = t.to(device=device(), dtype=torch.float64)
        return t.reshape(-1).contiguous().clone()
    import numpy as np
    arr = np.ascontiguousarray(np.asarray(values, dtype=float).reshape(-1))
    return torch.from_numpy(arr.copy()).to(device())
