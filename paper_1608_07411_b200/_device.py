"""Device-memory plumbing (torch is used only for allocation and streams)."""

from __future__ import annotations

import numpy as np
import torch

_NP2T = {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32,
         np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64,
         np.dtype(np.uint8): torch.uint8, np.dtype(np.bool_): torch.bool}
_T2NP = {v: k for k, v in _NP2T.items()}

# Reference pools put the first child block at slot 1 (octree.py:290,
# _kernels.pyx:37).  Offsetting every pool by 7 elements puts slot 1 -- and
# so every 8-slot block -- on a 32 B (fp32) / 64 B (fp64) boundary: one
# block of fp32 values is exactly one DRAM sector.
POOL_PAD = 7


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("a CUDA device is required (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def tdtype(dtype) -> torch.dtype:
    if isinstance(dtype, torch.dtype):
        return dtype
    return _NP2T[np.dtype(dtype)]


def npdtype(dtype) -> np.dtype:
    if isinstance(dtype, torch.dtype):
        return _T2NP[dtype]
    return np.dtype(dtype)


def pool_empty(cap: int, dtype, fill=None) -> torch.Tensor:
    """A device pool of ``cap`` slots whose slot 1 is sector aligned."""
    t = torch.empty(cap + POOL_PAD, dtype=tdtype(dtype), device=device())
    v = t[POOL_PAD:]
    if fill is not None:
        v.fill_(fill)
    return v


def to_pool(a, dtype=None, cap: int | None = None, fill=0) -> torch.Tensor:
    """Copy a host/device 1-D array into an aligned device pool."""
    if isinstance(a, torch.Tensor):
        src = a.to(device()) if dtype is None else a.to(device(), tdtype(dtype))
    else:
        arr = np.ascontiguousarray(a if dtype is None
                                   else np.asarray(a, dtype=npdtype(dtype)))
        src = torch.from_numpy(arr).to(device(), non_blocking=False)
    n = src.shape[0]
    cap = n if cap is None else max(cap, n)
    out = pool_empty(cap, src.dtype)
    out[:n].copy_(src)
    if cap > n:
        out[n:].fill_(fill)
    return out


def as_device(a, dtype=None) -> torch.Tensor:
    """Contiguous device tensor from numpy / torch input (no copy if already
    a matching contiguous device tensor)."""
    if isinstance(a, torch.Tensor):
        t = a if dtype is None else a.to(dtype=tdtype(dtype))
        t = t.to(device())
        return t.contiguous()
    arr = np.ascontiguousarray(np.asarray(a) if dtype is None
                               else np.asarray(a, dtype=npdtype(dtype)))
    return torch.from_numpy(arr).to(device())


def to_numpy(t) -> np.ndarray:
    if isinstance(t, torch.Tensor):
        return t.detach().cpu().numpy()
    return np.asarray(t)


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()
