"""CPU (gloo, world_size 2): the row-sharded apply's host logic — row
partition, padded all-gather and reassembly — with the oracle standing in for
each rank's device kernel. The N>1 GPU path differs only in the local kernel
(K2) and the backend (NCCL)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_1602_00001_b200.sharded import shard_rows


def test_shard_rows_partition():
    for N in (1, 7, 100, 16384, 16385):
        for G in (1, 2, 3, 8):
            spans = [shard_rows(N, G, r) for r in range(G)]
            assert spans[0][0] == 0
            for (a, n), (b, _) in zip(spans, spans[1:]):
                assert a + n == b
            assert sum(n for _, n in spans) == N
            assert max(n for _, n in spans) - min(n for _, n in spans) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, N, k, digits, seed, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import invop_oracle as O
        from paper_1602_00001_b200.sharded import ShardedApply, broadcast_rhs

        rng = np.random.default_rng(seed)
        X = torch.zeros((k, N), dtype=torch.float64)
        if rank == 0:
            X = torch.tensor(rng.standard_normal((k, N)))
        broadcast_rhs(X)
        row0, rows = shard_rows(N, world, rank)
        if digits is not None:
            # random mantissas: the oracle's ordered apply stands in for K2/K3
            mant = np.random.default_rng(seed + 1).integers(-3000, 3000, size=(N, N))

            def local(Xv, out, _m=mant[row0:row0 + rows]):
                out[:, :rows] = torch.tensor(O.ordered_apply(_m, digits, Xv.numpy()).reshape(k, rows))

            def full(Xv):
                return O.ordered_apply(mant, digits, Xv.numpy()).reshape(k, N)
        else:
            # structured operator (diagonal + all-ones) at sizes the dense
            # oracle cannot hold: y_ti = (i + 1) x_ti + sum_j x_tj
            def local(Xv, out):
                idx = torch.arange(row0, row0 + rows, dtype=torch.float64)
                out[:, :rows] = (idx + 1) * Xv[:, row0:row0 + rows] + Xv.sum(dim=1, keepdim=True)

            def full(Xv):
                idx = torch.arange(N, dtype=torch.float64)
                return ((idx + 1) * Xv + Xv.sum(dim=1, keepdim=True)).numpy()

        sh = ShardedApply(N, local, dtype=torch.float64, device=torch.device("cpu"))
        Y = sh.apply(X if k > 1 else X[0])
        out[rank] = Y.numpy().tobytes()
        if rank == 0:
            ref = full(X)
            out["ref"] = (ref if k > 1 else ref[0]).tobytes()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N,k,digits", [(64, 1, 3), (67, 1, 3), (67, 3, 3), (67, 64, 2),
                                        (16385, 1, None), (16385, 3, None), (16385, 64, None)])
def test_gloo_world2_matches_single(N, k, digits):
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, N, k, digits, 17, out), nprocs=world, join=True)
        assert out[0] == out["ref"]
        assert out[1] == out["ref"]


def test_row_offsets():
    from paper_1602_00001_b200.sharded import row_offsets

    for N, G in ((16385, 2), (67, 8), (100, 3)):
        off = row_offsets(N, G)
        assert off[0] == 0 and off[-1] == N
        assert all(off[r + 1] - off[r] == shard_rows(N, G, r)[1] for r in range(G))
