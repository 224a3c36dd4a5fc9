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


def _worker(rank, world, port, N, digits, seed, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import invop_oracle as O
        from paper_1602_00001_b200.sharded import ShardedApply, broadcast_rhs

        rng = np.random.default_rng(seed)
        mant = rng.integers(-3000, 3000, size=(N, N))
        x = torch.zeros(N, dtype=torch.float64)
        if rank == 0:
            x = torch.tensor(rng.standard_normal(N))
        broadcast_rhs(x)
        row0, rows = shard_rows(N, world, rank)

        def local(xv, _m=mant[row0:row0 + rows]):
            return torch.tensor(O.ordered_apply(_m, digits, xv.numpy()))

        sh = ShardedApply(N, local, dtype=torch.float64, device=torch.device("cpu"))
        y = sh.apply(x)
        out[rank] = y.numpy().tobytes()
        if rank == 0:
            out["ref"] = O.ordered_apply(mant, digits, x.numpy()).tobytes()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N", [64, 67])
def test_gloo_world2_matches_single(N):
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, N, 3, 17, out), nprocs=world, join=True)
        assert out[0] == out["ref"]
        assert out[1] == out["ref"]
