"""Skinned-body cases: device-side marker refresh
(update_samples, sampling.hpp:307-322) and tau_ext / CouplingStats reduction
(session.hpp:129-143), run by the oracle restatement and by the product.

The articulated koi, its forward kinematics (dynamics.hpp:23-61) and the
packed per-link pose come from paper_2206_01683_b200/scenes.py -- host-side
input generation, identical for both executors."""
from __future__ import annotations

import numpy as np

from oracle import bind as B
from paper_2206_01683_b200.scenes import Scene, koi_body


def skin_scene(dims=(48, 28, 28), dx=0.012, frame_mode="translation_yaw", bodies=1):
    origins = {1: [np.zeros(3)],
               2: [np.array([-0.27, 0.0, 0.0]), np.array([0.27, 0.0, 0.0])],
               3: [np.array([-0.5, 0.0, 0.0]), np.zeros(3), np.array([0.5, 0.0, 0.0])]}[bodies]
    return Scene("skin", dims, dx, frame_mode, [koi_body(dx) for _ in range(bodies)], 4,
                 origins=origins, motion="swim")


def init_fluid(sc, seed=41):
    n = sc.n_cells
    r = B.Rng(seed)
    rho = np.array([1.0 + 0.01 * (r.uniform() - 0.5) for _ in range(n)])
    u = np.array([0.01 * (r.uniform() - 0.5) for _ in range(3 * n)])
    return rho, u


def _frame_oracle(sc, k):
    f = sc.frame(k)
    return B.FrameState.make(p=f.p, pd=f.pd, pdd=f.pdd, q=f.q, omega=f.omega, alpha=f.alpha)


def run_oracle_skin(sc, steps, seed=41):
    """Per step: markers (pts, vel, nrm), fw, valid, tau per body, stats per body."""
    O = B.oracle()
    d = B.dims_arr(sc.dims)
    fm = {"none": 0, "translation": 1, "translation_yaw": 2, "full": 3}[sc.frame_mode]
    h = O.orc_session_create(B.iptr(d), sc.dx, sc.dt, sc.rho, sc.nu, 0, 0, 0, fm)
    rho, u = init_fluid(sc, seed)
    n = sc.n_cells
    f0 = np.empty(19 * n)
    O.orc_initialize(B.iptr(d), B.dptr(rho), B.dptr(u), B.dptr(f0))
    np.ctypeslib.as_array(O.orc_session_f(h), shape=(19 * n,))[:] = f0
    off, sks, rest, nrest, W, areas = sc.skin()
    nb = len(sks)
    m = int(off[-1])
    out = []
    for k in steps:
        O.orc_session_set_frame(h, _frame_oracle(sc, k))
        P = sc.poses(k)
        pts, vel, nrm = (np.empty((m, 3)) for _ in range(3))
        for b in range(nb):
            sl = slice(off[b], off[b + 1])
            pts[sl], vel[sl], nrm[sl] = B.skin_update(sks[b], P[b], rest[sl], nrest[sl], W[b])
        fw = np.zeros(3 * m)
        valid = np.zeros(m, np.int32)
        stats = np.zeros(7 * nb)
        fin = np.zeros(1, np.int32)
        mf = np.zeros(1)
        O.orc_session_step(h, nb, B.i64ptr(off), B.dptr(pts.reshape(-1)), B.dptr(vel.reshape(-1)),
                           B.dptr(nrm.reshape(-1)), B.dptr(np.ascontiguousarray(areas)), B.dptr(fw),
                           B.iptr(valid), B.dptr(stats), B.iptr(fin), B.dptr(mf))
        taus, st2 = [], []
        for b in range(nb):
            sl = slice(off[b], off[b + 1])
            t, s_ = B.skin_tau(sks[b], P[b], rest[sl], W[b], fw.reshape(-1, 3)[sl], valid[sl], vel[sl])
            taus.append(t)
            st2.append(s_)
        out.append(dict(pts=pts, vel=vel, nrm=nrm, fw=fw.reshape(-1, 3), valid=valid,
                        tau=np.concatenate(taus), stats=np.array(st2), stats_session=stats.reshape(-1, 7),
                        min_f=mf[0]))
    f = np.ctypeslib.as_array(O.orc_session_f(h), shape=(19 * n,)).copy()
    O.orc_session_destroy(h)
    return out, f


def run_gpu_skin(sc, steps, precision="fp64", seed=41):
    from paper_2206_01683_b200 import CoupledSession, SessionConfig
    s = CoupledSession(SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                                     frame_mode=sc.frame_mode, precision=precision,
                                     max_markers=sc.m))
    rho, u = init_fluid(sc, seed)
    s.initialize(rho, u)
    s.set_skin(*sc.skin())
    out = []
    for k in steps:
        s.set_frame(sc.frame(k))
        s.set_pose(sc.poses(k))
        st = s.step()
        pts, vel, nrm = s.markers()
        fw, valid, stats = s.marker_forces()
        taus, wst = s.body_wrench()
        out.append(dict(pts=pts, vel=vel, nrm=nrm, fw=fw, valid=valid, tau=np.concatenate(taus),
                        stats=wst, stats_session=stats, min_f=st.min_f, stencils=s.stencils()))
    f = s.get_f()
    s.close()
    return out, f
