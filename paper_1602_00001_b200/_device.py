"""Device plumbing: CUDA availability, streams and tensor transfer via torch.

PyTorch is used only to own device memory and streams; every computation on
the apply path runs in libinvop_b200.so. There is no CPU fallback: calling
into the device path without a CUDA device raises.
"""

from __future__ import annotations

import numpy as np

from .errors import InvopError

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as _t

        _torch = _t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise InvopError(
            "paper_1602_00001_b200 computes on a CUDA device (sm_100a); no GPU is visible "
            "and there is no CPU fallback"
        )
    return t


def stream_ptr() -> int:
    t = require_cuda()
    return t.cuda.current_stream().cuda_stream


def to_device(arr, dtype) -> "torch.Tensor":
    """Contiguous device tensor of `dtype` from numpy / list / tensor."""
    t = require_cuda()
    if isinstance(arr, t.Tensor):
        out = arr.to(device="cuda", dtype=dtype)
        return out.contiguous()
    np_dtype = {t.float64: np.float64, t.float32: np.float32, t.int64: np.int64,
                t.int32: np.int32, t.int8: np.int8}[dtype]
    a = np.ascontiguousarray(arr, dtype=np_dtype)
    if not a.flags.writeable:
        a = a.copy()
    return t.from_numpy(a).to("cuda", non_blocking=False)


def empty(shape, dtype) -> "torch.Tensor":
    t = require_cuda()
    return t.empty(shape, dtype=dtype, device="cuda")


def synchronize() -> None:
    require_cuda().cuda.synchronize()
