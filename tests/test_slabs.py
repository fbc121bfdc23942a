"""Multi-slab host logic on CPU (gloo, world sizes 2 and 3): partition, ring
neighbours, halo exchange placement, dt min-allreduce, fixed-order sums —
the same functions bench.py drives over NCCL on B200s."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2202_13821_b200 import slabs


def test_partition_covers_and_balances():
    for nz in (4, 7, 16, 128, 129):
        for w in (1, 2, 3, 4, 8):
            if nz < w:
                with pytest.raises(ValueError):
                    slabs.slab_partition(nz, w)
                continue
            p = slabs.slab_partition(nz, w)
            assert p[0][0] == 0
            assert sum(c for _, c in p) == nz
            for (b0, c0), (b1, _) in zip(p, p[1:]):
                assert b1 == b0 + c0
            assert max(c for _, c in p) - min(c for _, c in p) <= 1


def test_ring_neighbors():
    assert slabs.ring_neighbors(0, 4) == (3, 1)
    assert slabs.ring_neighbors(3, 4) == (2, 0)
    assert slabs.ring_neighbors(0, 2) == (1, 1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, L, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # a rank's packed boundary layers: bottom = 1000*rank + i, top = -(1000*rank + i)
        send_lo = torch.arange(L, dtype=torch.float64) + 1000 * rank
        send_hi = -(torch.arange(L, dtype=torch.float64) + 1000 * rank)
        recv_lo = torch.full((L,), np.nan, dtype=torch.float64)
        recv_hi = torch.full((L,), np.nan, dtype=torch.float64)
        slabs.exchange_halos(send_lo, send_hi, recv_lo, recv_hi, rank, world)
        lower, upper = slabs.ring_neighbors(rank, world)
        ok_lo = torch.equal(recv_lo, -(torch.arange(L, dtype=torch.float64) + 1000 * lower))  # lower's top
        ok_hi = torch.equal(recv_hi, torch.arange(L, dtype=torch.float64) + 1000 * upper)    # upper's bottom
        dmin = slabs.min_allreduce(1.0 + rank * 0.5 if rank != world - 1 else 0.25)
        sums = slabs.sum_allreduce([float(rank), 1.0])
        q.put((rank, ok_lo, ok_hi, dmin, sums))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_halo_exchange(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 50 * 16, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_lo, ok_hi, dmin, sums in res:
        assert ok_lo and ok_hi, rank
        assert dmin == 0.25
        assert sums == [float(sum(range(world))), float(world)]


def test_single_rank_exchange_is_periodic_wrap():
    L = 8
    send_lo, send_hi = torch.arange(L, dtype=torch.float64), -torch.arange(L, dtype=torch.float64)
    recv_lo, recv_hi = torch.zeros(L, dtype=torch.float64), torch.zeros(L, dtype=torch.float64)
    slabs.exchange_halos(send_lo, send_hi, recv_lo, recv_hi, 0, 1)
    assert torch.equal(recv_hi, send_lo) and torch.equal(recv_lo, send_hi)
