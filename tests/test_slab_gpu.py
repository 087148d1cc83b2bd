"""z-slab decomposition on the GPU: slabs exchanging their
boundary planes every step reproduce one monolithic session BIT-FOR-BIT, in
both precisions, with open and periodic z, an accelerating frame (global z in
the virtual force) and uneven slab depths.  The slabs run in one process on
one GPU with device copies standing in for the NCCL transfer (the transfer
routing itself is tested over gloo in test_slab_cpu.py)."""
import numpy as np
import pytest
import torch

import cases as K
from paper_2206_01683_b200 import CoupledSession, SessionConfig
from paper_2206_01683_b200.slab import SlabLayout, SlabRunner, device_views, split_field

pytestmark = pytest.mark.gpu

DT = 0.004


def _cfg(dims, prec, periodic, **kw):
    return SessionConfig(dims=dims, dx=0.01, dt=DT, rho=1000.0, nu=0.00089,
                         boundary="periodic" if periodic else "open",
                         frame_mode="translation_yaw", precision=prec, **kw)


def _init(dims, seed=7):
    n = int(np.prod(dims))
    r = np.random.default_rng(seed)
    return 1.0 + 0.01 * (r.random(n) - 0.5), 0.02 * (r.random(3 * n) - 0.5)


def _monolithic(dims, prec, periodic, steps):
    s = CoupledSession(_cfg(dims, prec, periodic))
    s.initialize(*_init(dims))
    for k in range(steps):
        s.set_frame(K._fs_to_product(K.frame_at(k, DT)))
        s.step_async()
    st = s.last_status()
    f = s.get_f().reshape(19, -1)
    s.close()
    return f, st


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
@pytest.mark.parametrize("periodic", [False, True])
def test_two_and_three_slabs_match_monolithic(prec, periodic):
    dims = (24, 20, 23)
    steps = 9
    ref, st_ref = _monolithic(dims, prec, periodic, steps)
    rho, u = _init(dims)
    for world in (2, 3):
        L = SlabLayout(dims[2], world, periodic)
        ss = []
        for r in range(world):
            z0, nz = L.planes(r)
            s = CoupledSession(_cfg((dims[0], dims[1], nz), prec, periodic, z_offset=z0,
                                    nz_global=dims[2]))
            s.initialize(split_field(rho, dims, L, r), split_field(u, dims, L, r, comps=3))
            ss.append(s)
        dt = "<f4" if prec == "fp32" else "<f8"
        views = [device_views(s, dt) for s in ss]  # (send_lo, send_hi, recv_lo, recv_hi)
        comm = torch.cuda.Stream()
        for k in range(steps):
            # fully asynchronous: the comm stream waits for every slab's packed
            # boundary planes, copies them across, and each slab waits for it
            for s in ss:
                s.set_frame(K._fs_to_product(K.frame_at(k, DT)))
                s.step_async()
                s.halo_begin(comm.cuda_stream)
            with torch.cuda.stream(comm):
                for r in range(world):
                    lo, hi = L.neighbours(r)
                    if lo is not None:
                        views[r][2].copy_(views[lo][1])
                    if hi is not None:
                        views[r][3].copy_(views[hi][0])
            for r, s in enumerate(ss):
                lo, hi = L.neighbours(r)
                s.halo_end(comm.cuda_stream, lo is not None, hi is not None)
        fs = [s.get_f().reshape(19, -1) for s in ss]
        sts = [s.last_status() for s in ss]
        got = np.concatenate(fs, axis=1)
        assert np.array_equal(got, ref), f"{world} slabs differ from the monolithic grid"
        assert min(st.min_f for st in sts) == st_ref.min_f
        for s in ss:
            s.close()


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_slab_runner_single_rank_periodic(prec):
    """SlabRunner on one rank is the plain (periodic) session."""
    dims = (16, 12, 10)
    steps = 6
    ref, _ = _monolithic(dims, prec, True, steps)
    L = SlabLayout(dims[2], 1, periodic=True)
    run = SlabRunner(dict(dims=dims, dx=0.01, dt=DT, rho=1000.0, nu=0.00089,
                          frame_mode="translation_yaw", precision=prec), L, 0)
    run.session.initialize(*_init(dims))
    for k in range(steps):
        run.session.set_frame(K._fs_to_product(K.frame_at(k, DT)))
        run.step_async()
    run.session.last_status()
    got = run.session.get_f().reshape(19, -1)
    run.close()
    assert np.array_equal(got, ref)


def test_markers_rejected_on_slab_sessions():
    s = CoupledSession(_cfg((16, 12, 6), "fp32", False, z_offset=4, nz_global=16))
    pts, nrm, area = K.fib_sphere(0.02, 10, np.zeros(3))
    with pytest.raises(Exception):
        s.set_markers(np.array([0, 10]), pts, np.zeros_like(pts), nrm, area)
    s.close()
