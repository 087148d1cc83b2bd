"""z-slab peer transport (fsg_peer_*): the halo exchange
inside the library -- the boundary planes' collision kernel stores the
crossing populations straight into the neighbours' halo planes, ordered by
stream memory operations on delivery counters.  Slabs stepped this way
reproduce one monolithic session BIT-FOR-BIT (open and periodic z, an
accelerating frame, uneven depths, a connect on a pulled state).

Two layouts run here on the one GPU a gpurun box has: several slab sessions
in one process (the neighbour's buffers are plain device pointers), and two
processes, each with its own slab session, connected through CUDA IPC
handles exchanged over a gloo process group -- the multi-process code path
of bench.py --gpus N, with both processes on device 0.  The ordering is
stream waits on memory, not spinning kernels, so ranks sharing a device
cannot deadlock each other."""
import os
import socket

import numpy as np
import pytest
import torch

import cases as K
from paper_2206_01683_b200 import CoupledSession, SessionConfig
from paper_2206_01683_b200.slab import SlabLayout, connect_peers, device_views, split_field

pytestmark = pytest.mark.gpu

DT = 0.004


def _cfg(dims, periodic, **kw):
    return SessionConfig(dims=dims, dx=0.01, dt=DT, rho=1000.0, nu=0.00089,
                         boundary="periodic" if periodic else "open",
                         frame_mode="translation_yaw", precision="fp32", **kw)


def _init(dims, seed=7):
    n = int(np.prod(dims))
    r = np.random.default_rng(seed)
    return 1.0 + 0.01 * (r.random(n) - 0.5), 0.02 * (r.random(3 * n) - 0.5)


def _monolithic(dims, periodic, steps):
    s = CoupledSession(_cfg(dims, periodic))
    s.initialize(*_init(dims))
    for k in range(steps):
        s.set_frame(K._fs_to_product(K.frame_at(k, DT)))
        s.step_async()
    st = s.last_status()
    f = s.get_f().reshape(19, -1)
    s.close()
    return f, st


def _slabs(dims, L, periodic):
    rho, u = _init(dims)
    ss = []
    for r in range(L.world):
        z0, nz = L.planes(r)
        s = CoupledSession(_cfg((dims[0], dims[1], nz), periodic, z_offset=z0, nz_global=dims[2]))
        s.initialize(split_field(rho, dims, L, r), split_field(u, dims, L, r, comps=3))
        ss.append(s)
    return ss


@pytest.mark.parametrize("periodic", [False, True])
@pytest.mark.parametrize("world", [2, 3])
def test_in_process_peer_slabs_match_monolithic(world, periodic):
    dims = (24, 20, 23)
    steps = 11
    ref, st_ref = _monolithic(dims, periodic, steps)
    L = SlabLayout(dims[2], world, periodic)
    ss = _slabs(dims, L, periodic)
    handles = [s.peer_export() for s in ss]
    for r, s in enumerate(ss):
        connect_peers(s, handles, L, r)
    for k in range(steps):
        for s in ss:  # each slab on its own stream; no host synchronisation
            s.set_frame(K._fs_to_product(K.frame_at(k, DT)))
            s.step_async()
    got = np.concatenate([s.get_f().reshape(19, -1) for s in ss], axis=1)
    sts = [s.last_status() for s in ss]
    torch.cuda.synchronize()
    for s in ss:
        s.close()
    assert np.array_equal(got, ref)
    assert min(st.min_f for st in sts) == st_ref.min_f


def test_connect_on_a_pulled_state_delivers_the_boundary_planes():
    """Two steps with the pack/copy transport, then peer-connect mid-run: the
    connect pushes the current boundary planes into the neighbours' halos."""
    dims, periodic, steps = (20, 16, 17), True, 9
    ref, _ = _monolithic(dims, periodic, steps)
    L = SlabLayout(dims[2], 3, periodic)
    ss = _slabs(dims, L, periodic)
    views = [device_views(s, "<f4") for s in ss]
    comm = torch.cuda.Stream()
    for k in range(2):
        for s in ss:
            s.set_frame(K._fs_to_product(K.frame_at(k, DT)))
            s.step_async()
            s.halo_begin(comm.cuda_stream)
        with torch.cuda.stream(comm):
            for r in range(3):
                lo, hi = L.neighbours(r)
                views[r][2].copy_(views[lo][1])
                views[r][3].copy_(views[hi][0])
        for s in ss:
            s.halo_end(comm.cuda_stream, True, True)
    torch.cuda.synchronize()
    handles = [s.peer_export() for s in ss]
    for r, s in enumerate(ss):
        connect_peers(s, handles, L, r)
    for k in range(2, steps):
        for s in ss:
            s.set_frame(K._fs_to_product(K.frame_at(k, DT)))
            s.step_async()
    got = np.concatenate([s.get_f().reshape(19, -1) for s in ss], axis=1)
    torch.cuda.synchronize()
    for s in ss:
        s.close()
    assert np.array_equal(got, ref)


def test_peer_connect_rejects_wrong_neighbours():
    dims = (16, 12, 12)
    L = SlabLayout(12, 3, False)
    ss = _slabs(dims, L, False)
    h = [s.peer_export() for s in ss]
    with pytest.raises(Exception):
        ss[0].peer_connect(None, h[2])  # not adjacent
    with pytest.raises(Exception):
        ss[1].peer_connect(b"\0" * 512, h[2])  # not a handle
    mono = CoupledSession(_cfg(dims, False))
    with pytest.raises(Exception):
        mono.peer_export()  # not a slab session
    mono.close()
    for s in ss:
        s.close()


# ------------------------------------------------- two processes, CUDA IPC --
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ipc_worker(rank, world, periodic, dims, steps, port, q):
    import torch.distributed as dist
    from paper_2206_01683_b200.slab import SlabRunner
    os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "8")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        L = SlabLayout(dims[2], world, periodic)
        run = SlabRunner(dict(dims=dims, dx=0.01, dt=DT, rho=1000.0, nu=0.00089,
                              frame_mode="translation_yaw", precision="fp32",
                              boundary="periodic" if periodic else "open"), L, rank)
        rho, u = _init(dims)
        run.session.initialize(split_field(rho, dims, L, rank), split_field(u, dims, L, rank, comps=3))
        for k in range(steps):
            run.session.set_frame(K._fs_to_product(K.frame_at(k, DT)))
            run.step_async()
        f = run.session.get_f().reshape(19, -1)
        st = run.session.last_status()
        q.put((rank, f, st.min_f, None))
        run.close()
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, None, None, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("periodic", [False, True])
def test_two_processes_ipc_match_monolithic(periodic):
    import torch.multiprocessing as mp
    dims, steps, world = (24, 20, 22), 10, 2
    ref, st_ref = _monolithic(dims, periodic, steps)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, periodic, dims, steps, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        r, f, mn, err = q.get(timeout=240)
        assert err is None, f"rank {r}: {err}"
        got[r] = (f, mn)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    f = np.concatenate([got[r][0] for r in range(world)], axis=1)
    assert np.array_equal(f, ref)
    assert min(got[r][1] for r in range(world)) == st_ref.min_f
