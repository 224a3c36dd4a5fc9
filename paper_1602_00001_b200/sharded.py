"""Row-sharded multi-GPU apply (one process per GPU, torch.distributed).

L^-1 is split into contiguous row blocks, one per rank; every rank builds
its own block on its own GPU (the block-LU constructor solves only for its
rows), so nothing of the operator crosses NVLink. An apply is

    y_r = L^-1[rows_r, :] rho      (K2 on rank r, no communication)
    y   = all_gather(y_0 .. y_{G-1})   (the one exchange step)

rho is either replicated by construction (same seed on every rank) or
broadcast once from rank 0. Uneven N is handled by padding the gathered
buffer to G * ceil(N/G) rows.

The same exchange is available below the Python layer for a C/C++ caller
that owns an ncclComm_t: `invop_apply_sharded` (include/invop_b200.h)
applies the local rows in place into the full y and exchanges the slices
with one NCCL group of in-place broadcasts (uneven shards, no padding).
"""

from __future__ import annotations

from typing import Callable, Optional

import numpy as np


def shard_rows(N: int, world: int, rank: int) -> tuple:
    """(row0, rows) of rank `rank`: contiguous, sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(N, world)
    row0 = rank * base + min(rank, extra)
    rows = base + (1 if rank < extra else 0)
    return row0, rows


class ShardedApply:
    """Row-sharded apply over a process group.

    `local_apply(x) -> y_shard` computes this rank's rows; by default it is
    the device fp32 kernel of a plan built from `stencil`. The exchange is
    one all_gather of fixed-size padded shards.
    """

    def __init__(self, N: int, local_apply: Callable, *, group=None, dtype=None, device=None):
        import torch
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.N = N
        self.row0, self.rows = shard_rows(N, self.world, self.rank)
        self.pad = -(-N // self.world)
        self.local_apply = local_apply
        self.dtype = dtype or torch.float32
        self.device = device or (torch.device("cuda", torch.cuda.current_device())
                                 if torch.cuda.is_available() else torch.device("cpu"))
        self._send = torch.zeros(self.pad, dtype=self.dtype, device=self.device)
        self._recv = torch.zeros(self.pad * self.world, dtype=self.dtype, device=self.device)
        self._counts = [shard_rows(N, self.world, r)[1] for r in range(self.world)]

    @classmethod
    def from_stencil(cls, stencil, digits: int, *, group=None, precision: str = "f32"):
        """Build this rank's block of the quantized L^-1 on its GPU (K4+K1)."""
        import torch
        import torch.distributed as dist

        from .dense import DeviceOperator
        from . import _lib as L

        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        row0, rows = shard_rows(stencil.n, world, rank)
        dplan = DeviceOperator(stencil).factor().quantized_rows(digits, row0, rows)
        mode = L.MODE_FAST if precision == "f32" else L.MODE_ORDERED
        dtype = torch.float32 if precision == "f32" else torch.float64

        def local(x, _p=dplan, _m=mode):
            return _p.apply_device(x, mode=_m)

        obj = cls(stencil.n, local, group=group, dtype=dtype)
        obj.plan = dplan
        return obj

    def apply(self, x):
        """Full y on every rank (device tensor when running on GPUs)."""
        y_local = self.local_apply(x)
        if self.world == 1:
            return y_local
        self._send[: self.rows].copy_(y_local.reshape(-1).to(self.dtype))
        if self._send.is_cuda:
            self.dist.all_gather_into_tensor(self._recv, self._send, group=self.group)
        else:
            parts = list(self._recv.view(self.world, self.pad).unbind(0))
            self.dist.all_gather(parts, self._send, group=self.group)
        if self.N % self.world == 0:
            return self._recv
        pieces = [self._recv[r * self.pad: r * self.pad + c] for r, c in enumerate(self._counts)]
        import torch

        return torch.cat(pieces)


def broadcast_rhs(x, src: int = 0, group=None):
    """rho from rank `src` to every rank (when it is not replicated by seed)."""
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(x, src=src, group=group)
    return x
