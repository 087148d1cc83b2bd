"""Canonical parity cases shared by the oracle tests, the golden-fixture
generator (tests/golden/make_golden.py) and the GPU parity tests.

Each case is a set of seeded inputs (arrays) plus a scripted sequence of
reference calls.  Three executors run the same script:

* ``run_ref``    -- the reference's own headers (oracle/_ref, this container)
* ``run_oracle`` -- the C restatement (oracle/liboracle.so)
* ``run_gpu``    -- the CUDA product through the C ABI (libfsg.so)

Inputs follow the reference tests' recipes (test_lattice.cpp, test_ib.cpp,
test_frame.cpp) with the seeds they use; the Rng is the reference's
xoshiro256** (core/rng.hpp), restated in oracle/bind.py and checked against
the compiled one.
"""
from __future__ import annotations

import math

import numpy as np

from oracle import bind as B

W = np.array([1 / 3] + [1 / 18] * 6 + [1 / 36] * 12)
EX = np.array([0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0])
EY = np.array([0, 0, 0, 1, -1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0, 1, -1, 1, -1])
EZ = np.array([0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1])


def feq_np(rho, u):
    """equilibrium (lattice.hpp:41-51) vectorised; rho[n], u[n,3] -> f[19*n]."""
    eu = np.outer(EX, u[:, 0]) + np.outer(EY, u[:, 1]) + np.outer(EZ, u[:, 2])
    u2 = (u * u).sum(1)
    return (W[:, None] * rho[None, :] * (1 + 3 * eu + 4.5 * eu * eu - 1.5 * u2[None, :])).reshape(-1)


def lattice_units(tau):
    """test_lattice.cpp:16-24: dx = dt = rho = 1, nu for tau."""
    return dict(dx=1.0, dt=1.0, rho=1.0, nu=(tau - 0.5) / 3.0)


# ----------------------------------------------------------------------------
def case_lbm_open():
    """test_lattice.cpp:313-333 recipe: 12^3 open, tau 0.8, Rng(3), F=(1e-5,2e-5,-1e-5)."""
    d = (12, 12, 12)
    n = int(np.prod(d))
    r = B.Rng(3)
    rho = np.empty(n)
    u = np.zeros((n, 3))
    for c in range(n):
        rho[c] = 1.0 + 0.02 * (r.uniform() - 0.5)
        u[c, 0] = 0.01 * r.uniform()
    F = np.tile([1e-5, 2e-5, -1e-5], n)
    return dict(name="lbm_open", dims=d, periodic=0, units=lattice_units(0.8), rho0=rho,
                u0=u.reshape(-1), F=F, steps=8)


def case_lbm_periodic():
    """test_lattice.cpp:164-187 recipe (10^3 periodic, Rng(7) + Rng(11) perturbation) with a
    random Guo force field added so the source term is exercised."""
    d = (10, 10, 10)
    n = int(np.prod(d))
    r = B.Rng(7)
    rho = np.empty(n)
    u = np.zeros((n, 3))
    for c in range(n):
        rho[c] = 1.0 + 0.05 * (r.uniform() - 0.5)
        u[c] = [r.uniform(-0.02, 0.02), r.uniform(-0.02, 0.02), r.uniform(-0.02, 0.02)]
    f0 = feq_np(rho, u)
    r2 = B.Rng(11)
    f0 = f0 * (1.0 + 0.01 * (r2.uniforms(19 * n) - 0.5))
    rf = B.Rng(13)
    F = 1e-4 * (rf.uniforms(3 * n) - 0.5)
    return dict(name="lbm_periodic", dims=d, periodic=1, units=lattice_units(0.8), f0=f0, F=F,
                steps=20)


def fib_sphere(radius, n, center):
    k = np.arange(n) + 0.5
    zc = 1.0 - 2.0 * k / n
    rr = np.sqrt(1.0 - zc * zc)
    ph = math.pi * (3.0 - math.sqrt(5.0)) * k
    nrm = np.stack([rr * np.cos(ph), rr * np.sin(ph), zc], axis=1)
    return center + radius * nrm, nrm, np.full(n, 4 * math.pi * radius * radius / n)


def frame_at(step, dt):
    """A prescribed accelerating, yawing frame (all VF terms non-zero)."""
    t = step * dt
    yaw = 0.3 + 0.2 * math.sin(3.0 * t)
    return B.FrameState.make(
        p=(0.01 * t, -0.005, 0.002), pd=(0.05 + 0.01 * math.cos(3 * t), 0.0, 0.001),
        pdd=(0.3 * math.sin(5 * t), -0.1, 0.05),
        q=(math.cos(0.5 * yaw), 0.0, 0.0, math.sin(0.5 * yaw)),
        omega=(0.02, -0.01, 0.6 * math.cos(3.0 * t)), alpha=(0.05, 0.01, -1.8 * math.sin(3.0 * t)))


def case_session_frame():
    """Coupled step (session.hpp:94-166) in an accelerating, rotating frame:
    20x16x16 open box, dx 0.01, Peskin4, slip; an oscillating sphere of
    markers (some pushed out of bounds); 4 steps, recenter(1,0,-1), 2 steps."""
    d = (20, 16, 16)
    n = int(np.prod(d))
    r = B.Rng(21)
    rho = np.array([1.0 + 0.01 * (r.uniform() - 0.5) for _ in range(n)])
    u = np.array([[0.01 * (r.uniform() - 0.5) for _ in range(3)] for _ in range(n)])
    pts0, nrm, area = fib_sphere(0.035, 160, np.array([0.003, -0.002, 0.001]))
    # a few markers placed outside the kernel margin (counted as out of bounds)
    pts0[:3] += np.array([0.09, 0.0, 0.0])
    script = [("step", k) for k in range(4)] + [("recenter", (1, 0, -1))] + \
             [("step", k) for k in range(4, 6)]
    return dict(name="session_frame", dims=d, periodic=0,
                units=dict(dx=0.01, dt=0.004, rho=1000.0, nu=0.00089), kernel=0, wall=0,
                frame_mode=2, rho0=rho, u0=u.reshape(-1), pts0=pts0, nrm=nrm, area=area,
                offsets=np.array([0, len(area)], dtype=np.int64), script=script)


def case_session_roma3():
    """Two bodies, Roma3 kernel, no-slip wall, frame None (fixed domain)."""
    d = (18, 16, 14)
    n = int(np.prod(d))
    r = B.Rng(33)
    rho = np.array([1.0 + 0.01 * (r.uniform() - 0.5) for _ in range(n)])
    u = np.array([[0.02 * (r.uniform() - 0.5) for _ in range(3)] for _ in range(n)])
    p1, n1, a1 = fib_sphere(0.025, 90, np.array([-0.035, 0.0, 0.0]))
    p2, n2, a2 = fib_sphere(0.02, 60, np.array([0.04, 0.01, -0.005]))
    return dict(name="session_roma3", dims=d, periodic=0,
                units=dict(dx=0.01, dt=0.004, rho=1000.0, nu=0.00089), kernel=1, wall=1,
                frame_mode=0, rho0=rho, u0=u.reshape(-1), pts0=np.concatenate([p1, p2]),
                nrm=np.concatenate([n1, n2]), area=np.concatenate([a1, a2]),
                offsets=np.array([0, 90, 150], dtype=np.int64),
                script=[("step", k) for k in range(3)])


def case_recenter():
    """test_frame.cpp:114-159 recipe: 12x10x9, Rng(5)."""
    d = (12, 10, 9)
    n = int(np.prod(d))
    r = B.Rng(5)
    rho = np.empty(n)
    u = np.zeros((n, 3))
    for c in range(n):
        rho[c] = 1.0 + 0.01 * r.uniform()
        u[c, 0] = 0.01 * r.uniform()
    return dict(name="recenter", dims=d, f0=feq_np(rho, u), shifts=[(1, 0, 0), (-2, 1, 3)],
                units=dict(dx=0.02, dt=0.004, rho=1000.0, nu=0.00089))


def marker_state(case, step):
    """World-frame marker state of a session case at `step` (prescribed motion)."""
    dt = case["units"]["dt"]
    t = step * dt
    shift = np.array([0.004 * math.sin(20 * t), 0.002 * math.cos(15 * t), 0.0])
    shift = shift + np.asarray(case.get("jumps", {}).get(step, (0.0, 0.0, 0.0)))  # teleports
    vel = np.tile([0.08 * math.cos(20 * t), -0.03 * math.sin(15 * t), 0.01], (len(case["area"]), 1))
    return (np.ascontiguousarray(case["pts0"] + shift), np.ascontiguousarray(vel),
            np.ascontiguousarray(case["nrm"]), np.ascontiguousarray(case["area"]))


# ----------------------------------------------------------------------------
# executors
def run_ref_lbm(case):
    R = B.ref()
    d = case["dims"]
    un = case["units"]
    h = R.ref_session_create(*d, un["dx"], un["dt"], un["rho"], un["nu"], case["periodic"], 0, 0, 0)
    if "f0" in case:
        R.ref_set_f(h, B.dptr(np.ascontiguousarray(case["f0"])))
    else:
        R.ref_initialize(h, B.dptr(case["rho0"]), B.dptr(case["u0"]))
    R.ref_set_force(h, B.dptr(np.ascontiguousarray(case["F"])))
    mins, fins = [], []
    for _ in range(case["steps"]):
        fin = np.zeros(1, np.int32)
        mf = np.zeros(1)
        R.ref_collide_and_stream(h, B.iptr(fin), B.dptr(mf))
        mins.append(mf[0])
        fins.append(fin[0])
    n = int(np.prod(d))
    f = np.empty(19 * n)
    R.ref_get_f(h, B.dptr(f))
    rho = np.empty(n)
    u = np.empty(3 * n)
    nonpos = R.ref_macroscopic(h, B.dptr(rho), B.dptr(u))
    mass = R.ref_total_mass(h)
    mom = np.zeros(3)
    R.ref_total_momentum(h, B.dptr(mom))
    R.ref_session_destroy(h)
    return dict(f=f, min_f=np.array(mins), finite=np.array(fins), rho=rho, u=u, nonpos=nonpos,
                mass=mass, momentum=mom)


def run_oracle_lbm(case):
    O = B.oracle()
    d = B.dims_arr(case["dims"])
    n = int(np.prod(case["dims"]))
    un = case["units"]
    tau = O.orc_tau(un["dx"], un["dt"], un["nu"])
    if "f0" in case:
        fa = np.array(case["f0"], dtype=np.float64)
    else:
        fa = np.empty(19 * n)
        O.orc_initialize(B.iptr(d), B.dptr(case["rho0"]), B.dptr(case["u0"]), B.dptr(fa))
    fb = np.empty_like(fa)
    F = np.ascontiguousarray(case["F"])
    mins, fins = [], []
    for _ in range(case["steps"]):
        fin = np.zeros(1, np.int32)
        mf = np.zeros(1)
        O.orc_collide_and_stream(B.iptr(d), case["periodic"], tau, B.dptr(fa), B.dptr(fb),
                                 B.dptr(F), B.iptr(fin), B.dptr(mf))
        fa, fb = fb, fa
        mins.append(mf[0])
        fins.append(fin[0])
    rho = np.empty(n)
    u = np.empty(3 * n)
    nonpos = O.orc_macroscopic(B.iptr(d), B.dptr(fa), B.dptr(F), B.dptr(rho), B.dptr(u))
    mom = np.zeros(3)
    O.orc_total_momentum(B.iptr(d), B.dptr(fa), B.dptr(mom))
    return dict(f=fa, min_f=np.array(mins), finite=np.array(fins), rho=rho, u=u, nonpos=nonpos,
                mass=O.orc_total_mass(B.iptr(d), B.dptr(fa)), momentum=mom)


def _session_outputs_init(case):
    return dict(min_f=[], finite=[], nonpos=[], oob=[])


def run_ref_session(case):
    R = B.ref()
    d = case["dims"]
    un = case["units"]
    n = int(np.prod(d))
    h = R.ref_session_create(*d, un["dx"], un["dt"], un["rho"], un["nu"], case["periodic"],
                             case["kernel"], case["wall"], case["frame_mode"])
    R.ref_initialize(h, B.dptr(case["rho0"]), B.dptr(case["u0"]))
    out = _session_outputs_init(case)
    m = len(case["area"])
    nb = len(case["offsets"]) - 1
    for op, arg in case["script"]:
        if op == "recenter":
            R.ref_recenter(h, B.iptr(np.array(arg, dtype=np.int32)))
            p = np.zeros(3)
            R.ref_get_frame_p(h, B.dptr(p))
            out["frame_p_rc"] = p
            continue
        fs = frame_at(arg, un["dt"]) if case["frame_mode"] else B.FrameState.make()
        R.ref_set_frame(h, *(B.dptr(np.array(list(getattr(fs, k)))) for k in
                             ("p", "pd", "pdd", "q", "omega", "alpha")))
        pts, vel, nrm, area = marker_state(case, arg)
        fw = np.zeros(3 * m)
        valid = np.zeros(m, np.int32)
        stats = np.zeros(7 * nb)
        fin = np.zeros(1, np.int32)
        mf = np.zeros(1)
        nonpos = R.ref_session_step(h, nb, B.i64ptr(case["offsets"]), B.dptr(pts.reshape(-1)),
                                    B.dptr(vel.reshape(-1)), B.dptr(nrm.reshape(-1)), B.dptr(area),
                                    B.dptr(fw), B.iptr(valid), B.dptr(stats), B.iptr(fin), B.dptr(mf))
        xl = np.zeros(3 * m)
        R.ref_session_marker_xlat(h, m, B.dptr(pts.reshape(-1)), B.dptr(xl))
        out["min_f"].append(mf[0])
        out["finite"].append(fin[0])
        out["nonpos"].append(nonpos)
        out["oob"].append(int((valid == 0).sum()))
        last = dict(fw=fw, valid=valid, stats=stats, xl=xl)
    f = np.empty(19 * n)
    R.ref_get_f(h, B.dptr(f))
    rho = np.empty(n)
    u = np.empty(3 * n)
    R.ref_get_macro(h, B.dptr(rho), B.dptr(u))
    F = np.empty(3 * n)
    R.ref_get_force(h, B.dptr(F))
    R.ref_session_destroy(h)
    # stencil ranges of the last step (kernel.hpp:36-40) from the reference's own range()
    lo_hi = np.zeros((m, 6), np.int32)
    for i in range(m):
        if last["valid"][i]:
            for a in range(3):
                lo = np.zeros(1, np.int32)
                hi = np.zeros(1, np.int32)
                R.ref_range(case["kernel"], last["xl"][3 * i + a], B.iptr(lo), B.iptr(hi))
                lo_hi[i, a], lo_hi[i, 3 + a] = lo[0], hi[0]
        else:
            lo_hi[i, 3:] = -1
    return dict(f=f, rho=rho, u=u, F=F, fw=last["fw"], valid=last["valid"], stats=last["stats"],
                stencils=lo_hi, frame_p_rc=out.get("frame_p_rc", np.zeros(3)), min_f=np.array(out["min_f"]),
                finite=np.array(out["finite"]), nonpos=np.array(out["nonpos"]),
                oob=np.array(out["oob"]))


def run_oracle_session(case):
    O = B.oracle()
    d = B.dims_arr(case["dims"])
    un = case["units"]
    n = int(np.prod(case["dims"]))
    h = O.orc_session_create(B.iptr(d), un["dx"], un["dt"], un["rho"], un["nu"], case["periodic"],
                             case["kernel"], case["wall"], case["frame_mode"])
    f0 = np.empty(19 * n)
    O.orc_initialize(B.iptr(d), B.dptr(case["rho0"]), B.dptr(case["u0"]), B.dptr(f0))
    np.ctypeslib.as_array(O.orc_session_f(h), shape=(19 * n,))[:] = f0
    out = _session_outputs_init(case)
    m = len(case["area"])
    nb = len(case["offsets"]) - 1
    for op, arg in case["script"]:
        if op == "recenter":
            O.orc_session_recenter(h, B.iptr(np.array(arg, dtype=np.int32)))
            cur = B.FrameState()
            O.orc_session_get_frame(h, cur)
            out["frame_p_rc"] = np.array(list(cur.p))
            continue
        fs = frame_at(arg, un["dt"]) if case["frame_mode"] else B.FrameState.make()
        O.orc_session_set_frame(h, fs)
        pts, vel, nrm, area = marker_state(case, arg)
        fw = np.zeros(3 * m)
        valid = np.zeros(m, np.int32)
        stats = np.zeros(7 * nb)
        fin = np.zeros(1, np.int32)
        mf = np.zeros(1)
        nonpos = O.orc_session_step(h, nb, B.i64ptr(case["offsets"]), B.dptr(pts.reshape(-1)),
                                    B.dptr(vel.reshape(-1)), B.dptr(nrm.reshape(-1)), B.dptr(area),
                                    B.dptr(fw), B.iptr(valid), B.dptr(stats), B.iptr(fin), B.dptr(mf))
        out["min_f"].append(mf[0])
        out["finite"].append(fin[0])
        out["nonpos"].append(nonpos)
        out["oob"].append(int((valid == 0).sum()))
        last = dict(fw=fw, valid=valid, stats=stats)
    f = np.ctypeslib.as_array(O.orc_session_f(h), shape=(19 * n,)).copy()
    F = np.ctypeslib.as_array(O.orc_session_force(h), shape=(3 * n,)).copy()
    rho = np.ctypeslib.as_array(O.orc_session_rho(h), shape=(n,)).copy()
    u = np.ctypeslib.as_array(O.orc_session_u(h), shape=(3 * n,)).copy()
    O.orc_session_destroy(h)
    return dict(f=f, rho=rho, u=u, F=F, fw=last["fw"], valid=last["valid"], stats=last["stats"],
                frame_p_rc=out.get("frame_p_rc", np.zeros(3)), min_f=np.array(out["min_f"]),
                finite=np.array(out["finite"]), nonpos=np.array(out["nonpos"]),
                oob=np.array(out["oob"]))



# ----------------------------------------------------------------------------
# GPU executors (the product, through the C ABI)
def _gpu_cfg(case, precision, **kw):
    from paper_2206_01683_b200 import SessionConfig
    un = case["units"]
    frame = {0: "none", 1: "translation", 2: "translation_yaw", 3: "full"}[case.get("frame_mode", 0)]
    return SessionConfig(dims=case["dims"], dx=un["dx"], dt=un["dt"], rho=un["rho"], nu=un["nu"],
                         boundary="periodic" if case.get("periodic") else "open",
                         kernel=["peskin4", "roma3"][case.get("kernel", 0)],
                         wall=["slip", "noslip"][case.get("wall", 0)], frame_mode=frame,
                         precision=precision, **kw)


def _fs_to_product(fs):
    from paper_2206_01683_b200 import FrameState
    return FrameState(*(np.array(list(getattr(fs, k))) for k in
                        ("p", "pd", "pdd", "q", "omega", "alpha")))


def run_gpu_lbm(case, precision="fp64"):
    from paper_2206_01683_b200 import CoupledSession
    s = CoupledSession(_gpu_cfg(case, precision))
    if "f0" in case:
        s.set_f(case["f0"])
    else:
        s.initialize(case["rho0"], case["u0"])
    s.set_force(case["F"])
    mins, fins = [], []
    for _ in range(case["steps"]):
        st = s.collide_and_stream()
        mins.append(st.min_f)
        fins.append(int(st.finite))
    f = s.get_f()
    rho, u, nonpos = s.macroscopic()
    out = dict(f=f, min_f=np.array(mins), finite=np.array(fins), rho=rho, u=u.reshape(-1),
               nonpos=nonpos, mass=s.total_mass(), momentum=s.total_momentum())
    s.close()
    return out


def run_gpu_session(case, precision="fp64"):
    from paper_2206_01683_b200 import CoupledSession
    un = case["units"]
    s = CoupledSession(_gpu_cfg(case, precision))
    s.initialize(case["rho0"], case["u0"])
    out = _session_outputs_init(case)
    for op, arg in case["script"]:
        if op == "recenter":
            s.recenter(arg)
            out["frame_p_rc"] = s.frame_state().p.copy()
            continue
        fs = frame_at(arg, un["dt"]) if case["frame_mode"] else B.FrameState.make()
        s.set_frame(_fs_to_product(fs))
        s.set_markers(case["offsets"], *marker_state(case, arg))
        st = s.step()
        out["min_f"].append(st.min_f)
        out["finite"].append(int(st.finite))
        out["nonpos"].append(st.n_nonpositive_rho)
        out["oob"].append(st.out_of_bounds_markers)
    fw, valid, stats = s.marker_forces()
    rho, u = s.macro()
    res = dict(f=s.get_f(), rho=rho, u=u.reshape(-1), F=s.force().reshape(-1), fw=fw.reshape(-1),
               valid=valid, stats=stats.reshape(-1), stencils=s.stencils(),
               frame_p_rc=out.get("frame_p_rc", np.zeros(3)), min_f=np.array(out["min_f"]),
               finite=np.array(out["finite"]), nonpos=np.array(out["nonpos"]),
               oob=np.array(out["oob"]))
    s.close()
    return res


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64).reshape(-1)
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# ----------------------------------------------------------------------------
# FrameFollower (frame.hpp:70-125): a robot-base target trajectory with
# translation, yaw, pitch and roll, two resets, 240 steps of dt = 0.004
FOLLOW_MODES = ("none", "translation", "translation_yaw", "full")


def follower_script():
    ops = [("reset", (0.01, -0.02, 0.005), 0.3)]
    for k in range(240):
        t = 0.004 * k
        yaw = 0.3 + 1.9 * math.sin(2.1 * t) + (3.0 if k > 150 else 0.0)  # crosses +-pi
        pitch, roll = 0.25 * math.sin(3.3 * t), 0.2 * math.cos(2.7 * t)
        cy, sy = math.cos(0.5 * yaw), math.sin(0.5 * yaw)
        cp, sp = math.cos(0.5 * pitch), math.sin(0.5 * pitch)
        cr, sr = math.cos(0.5 * roll), math.sin(0.5 * roll)
        q = (cy * cp * cr + sy * sp * sr, cy * cp * sr - sy * sp * cr,
             cy * sp * cr + sy * cp * sr, sy * cp * cr - cy * sp * sr)  # ZYX
        p = (0.1 * t + 0.02 * math.sin(7 * t), 0.03 * math.cos(5 * t), 0.01 * math.sin(3 * t))
        ops.append(("step", p, q))
        if k == 120:
            ops.append(("reset", (0.2, 0.0, -0.01), -2.5))
    return ops


def run_ref_follower(mode, ops, tc=0.2):
    """-> [n_states, 19] (p, pd, pdd, q(w,x,y,z), omega, alpha) after every op."""
    R = B.ref()
    h = R.ref_follower_create(FOLLOW_MODES.index(mode), tc)
    out, buf = [], np.zeros(22)
    for op in ops:
        if op[0] == "reset":
            R.ref_follower_reset(h, B.dptr(np.array(op[1], dtype=np.float64)), op[2])
        else:
            R.ref_follower_step(h, B.dptr(np.array(op[1], dtype=np.float64)),
                                B.dptr(np.array(op[2], dtype=np.float64)), 0.004)
        R.ref_follower_state(h, B.dptr(buf))
        out.append(buf[:19].copy())
    R.ref_follower_destroy(h)
    return np.array(out)


def run_product_follower(mode, ops, tc=0.2):
    from paper_2206_01683_b200 import FrameFollower
    f = FrameFollower(mode, tc)
    out = []
    for op in ops:
        if op[0] == "reset":
            f.reset(op[1], op[2])
        else:
            f.step(op[1], op[2], 0.004)
        s = f.state()
        out.append(np.concatenate([s.p, s.pd, s.pdd, s.q, s.omega, s.alpha]))
    f.close()
    return np.array(out)
