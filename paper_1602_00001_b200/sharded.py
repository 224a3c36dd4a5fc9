"""Row-sharded multi-GPU apply (one process per GPU, torch.distributed).

L^-1 is split into contiguous row blocks, one per rank; every rank builds
its own block on its own GPU (the block-LU constructor solves only for its
rows), so nothing of the operator crosses NVLink. An apply of k right-hand
sides X [k, N] is

    Y_r = L^-1[rows_r, :] X^T        (K2 / K3 on rank r, no communication)
    Y   = all_gather(Y_0 .. Y_{G-1})  (the one exchange step)

Each rank writes its rows straight into its slice of a staging buffer
[world][k][pad] (pad = the largest shard), ONE all_gather_into_tensor fills
every slice, and one kernel (`invop_unshard`) scatters the slices into
Y [k, N] — uneven N included. The reference apply is 1-D only
(/root/reference/pkg/src/invop/applyplan.py:178-180); rows are independent,
so the sharded result equals the single-GPU result bit for bit.

rho is either replicated by construction (same seed on every rank) or
broadcast once from rank 0 (`broadcast_rhs`).

The same exchange is available below the Python layer for a C/C++ caller
that owns an ncclComm_t: `invop_apply_sharded` (include/invop_b200.h).
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


def row_offsets(N: int, world: int) -> np.ndarray:
    """int64 [world + 1]: rank r owns rows [off[r], off[r+1])."""
    off = np.zeros(world + 1, dtype=np.int64)
    for r in range(world):
        off[r + 1] = off[r] + shard_rows(N, world, r)[1]
    return off


class ShardedApply:
    """Row-sharded apply over a process group.

    `local_apply(X, out)` computes this rank's rows of X [k, N] into `out`, a
    [k, pad] view whose first `rows` columns it must fill (extra columns are
    padding); by default it is the device kernel of a plan built from
    `stencil` (`from_stencil`). `apply` accepts x [N] or X [k, N] and returns
    the full y [N] / Y [k, N] on every rank.
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
        self.offsets = row_offsets(N, self.world)
        self.local_apply = local_apply
        self.dtype = dtype or torch.float32
        self.device = device or (torch.device("cuda", torch.cuda.current_device())
                                 if torch.cuda.is_available() else torch.device("cpu"))
        self._stage = None

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

        def local(X, out, _p=dplan, _m=mode):
            _p.apply_device(X, out, ldy=out.stride(0), mode=_m)

        obj = cls(stencil.n, local, group=group, dtype=dtype)
        obj.plan = dplan
        return obj

    def _staging(self, k: int):
        import torch

        if self._stage is None or self._stage.shape[1] != k:
            self._stage = torch.zeros((self.world, k, self.pad), dtype=self.dtype, device=self.device)
        return self._stage

    def apply(self, x):
        """Full y on every rank (device tensor when running on GPUs)."""
        import torch

        one = x.dim() == 1
        X = x.reshape(1, -1) if one else x
        if X.shape[1] != self.N:
            raise ValueError("vector length %d does not match n=%d" % (X.shape[1], self.N))
        k = X.shape[0]
        stage = self._staging(k)
        mine = stage[self.rank]                        # [k, pad]
        self.local_apply(X, mine)
        if self.world > 1:
            if stage.is_cuda:
                self.dist.all_gather_into_tensor(stage.view(-1), mine.reshape(-1), group=self.group)
            else:
                parts = list(stage.view(self.world, -1).unbind(0))
                self.dist.all_gather(parts, mine.reshape(-1).clone(), group=self.group)
        Y = torch.empty((k, self.N), dtype=self.dtype, device=self.device)
        if stage.is_cuda:
            import ctypes as C

            from . import _device as dev
            from . import _lib as L

            offs = np.ascontiguousarray(self.offsets)
            L.check(L.lib.invop_unshard(stage.data_ptr(), self.world, offs.ctypes.data, k, self.pad,
                                        Y.data_ptr(), self.N,
                                        L.F64 if self.dtype == torch.float64 else L.F32,
                                        C.c_void_p(dev.stream_ptr())), "unshard")
        else:
            # host logic of the same reassembly (CPU process groups in the tests)
            for r in range(self.world):
                a, b = int(self.offsets[r]), int(self.offsets[r + 1])
                Y[:, a:b] = stage[r, :, : b - a]
        return Y.view(-1) if one else Y


def broadcast_rhs(x, src: int = 0, group=None):
    """rho from rank `src` to every rank (when it is not replicated by seed)."""
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(x, src=src, group=group)
    return x
