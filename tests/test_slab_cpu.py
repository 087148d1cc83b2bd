"""Host-side z-slab logic on CPUs: the layout, and the
halo exchange itself across world_size 2 and 3 gloo process groups -- the
same `exchange` the GPU run drives over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2206_01683_b200.slab import SlabLayout, exchange, split_field


def test_layout_partitions_and_neighbours():
    L = SlabLayout(10, 3)
    assert [L.planes(r) for r in range(3)] == [(0, 4), (4, 3), (7, 3)]
    assert [L.neighbours(r) for r in range(3)] == [(None, 1), (0, 2), (1, None)]
    P = SlabLayout(512, 8, periodic=True)
    assert sum(P.planes(r)[1] for r in range(8)) == 512
    assert P.neighbours(0) == (7, 1) and P.neighbours(7) == (6, 0)
    with pytest.raises(ValueError):
        SlabLayout(5, 4).validate()  # a slab of one plane cannot clamp locally


def test_split_field_matches_global_order():
    dims = (3, 2, 7)
    L = SlabLayout(7, 2)
    g = np.arange(np.prod(dims) * 3, dtype=np.float64)
    parts = [split_field(g, dims, L, r, comps=3) for r in range(2)]
    assert np.array_equal(np.concatenate(parts), g)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, periodic, port, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    L = SlabLayout(4 * world, world, periodic)
    n = 5 * 6  # 5 populations x a 3x2 plane
    send_lo = torch.arange(n, dtype=torch.float32) + 1000 * rank + 100
    send_hi = torch.arange(n, dtype=torch.float32) + 1000 * rank + 200
    recv_lo = torch.full((n,), -1.0)
    recv_hi = torch.full((n,), -1.0)
    have = exchange(send_lo, send_hi, recv_lo, recv_hi, rank, L)
    q.put((rank, have, recv_lo.numpy().copy(), recv_hi.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,periodic", [(2, False), (2, True), (3, False), (3, True)])
def test_exchange_gloo(world, periodic):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, periodic, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        r, have, lo, hi = q.get(timeout=120)
        got[r] = (have, lo, hi)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    L = SlabLayout(4 * world, world, periodic)
    n = 30
    for r in range(world):
        (have_lo, have_hi), lo, hi = got[r]
        nl, nh = L.neighbours(r)
        assert have_lo == (nl is not None) and have_hi == (nh is not None)
        # the lower neighbour's top face arrives in recv_lo, the upper's bottom in recv_hi
        if nl is not None:
            assert np.array_equal(lo, np.arange(n) + 1000 * nl + 200)
        else:
            assert np.all(lo == -1)
        if nh is not None:
            assert np.array_equal(hi, np.arange(n) + 1000 * nh + 100)
        else:
            assert np.all(hi == -1)
