"""Long-horizon parity of the fp32 throughput path (north_star: fp32 density,
velocity and body force within rel-L2 <= 1e-5 "after N steps").

The BASELINE scenes run their full step counts (c1 1000 steps -- the
CPU-runnable oracle case --, c2 1000, c3 500, c5 1000) on identical
prescribed inputs in throughput mode (fp32 deviations, the benchmarked
kernels) and in parity mode (fp64, bit-exact to the reference: see
test_parity_gpu.py); c1 is also run through the reference itself
(oracle/_ref: the reference headers compiled unmodified, OpenMP on the host)
and compared bit for bit with parity mode and within tolerance with
throughput mode.  Every 100 steps the marker stencil index sets and validity
must be identical.  The fp32 body force compared is the field the collision
kernel consumed (fsg_set_force_capture), not a rebuild.

Reference path: solver.hpp:103-178 driven by session.hpp:87-166.
"""
import numpy as np
import pytest

import cases as K

pytestmark = pytest.mark.gpu

TOL32 = 1e-5  # rel-L2, north_star


def _session(sc, prec):
    from paper_2206_01683_b200 import CoupledSession, SessionConfig
    s = CoupledSession(SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                                     frame_mode=sc.frame_mode, precision=prec,
                                     max_markers=sc.m))
    if prec == "fp32":
        s.set_force_capture(True)
    return s


def _fields(s):
    fw, valid, _ = s.marker_forces()
    rho, u = s.macro()
    return dict(rho=rho, u=u, F=s.force(), fw=fw, valid=valid, st=s.stencils())


def _run_pair(name, steps, check_every=100):
    from paper_2206_01683_b200.scenes import make_scene
    sc = make_scene(name)
    ss = {p: _session(sc, p) for p in ("fp64", "fp32")}
    for k in range(steps):
        fr, mk = sc.frame(k), sc.markers(k)
        for p, s in ss.items():
            s.set_frame(fr)
            s.set_markers(sc.offsets, *mk)
            st = s.step()
            assert st.stable(), (name, p, k)
        if (k + 1) % check_every == 0:
            st64, st32 = ss["fp64"].stencils(), ss["fp32"].stencils()
            assert np.array_equal(st64, st32), (name, k + 1)
            v64 = ss["fp64"].marker_forces()[1]
            v32 = ss["fp32"].marker_forces()[1]
            assert np.array_equal(v64, v32), (name, k + 1)
    out = {p: _fields(s) for p, s in ss.items()}
    for s in ss.values():
        s.close()
    return sc, out


def _assert_tol(a, b, what):
    errs = {
        "rho-1": K.rel_l2(a["rho"] - 1.0, b["rho"] - 1.0),
        "u": K.rel_l2(a["u"], b["u"]),
        "F": K.rel_l2(a["F"], b["F"]),
        "fw": K.rel_l2(a["fw"], b["fw"]),
    }
    bad = {k: v for k, v in errs.items() if not v <= TOL32}
    assert not bad, f"{what}: rel-L2 over {TOL32}: {bad} (all: {errs})"
    assert np.array_equal(a["st"], b["st"]) and np.array_equal(a["valid"], b["valid"]), what
    return errs


@pytest.mark.parametrize("name,steps", [("c2", 1000), ("c3", 500), ("c5", 1000)])
def test_scene_fp32_vs_fp64_full_length(name, steps):
    _, out = _run_pair(name, steps)
    _assert_tol(out["fp32"], out["fp64"], f"{name} after {steps} steps")


def _run_reference_c1(sc, steps):
    """The reference's own code (oracle/_ref) on the host: c1 for `steps`
    coupled steps; returns (rho, u, F, fw, valid)."""
    from oracle import bind as B
    R = B.ref()
    fm = {"none": 0, "translation": 1, "translation_yaw": 2, "full": 3}[sc.frame_mode]
    h = R.ref_session_create(*sc.dims, sc.dx, sc.dt, sc.rho, sc.nu, 0, 0, 0, fm)
    m, nb = sc.m, len(sc.bodies)
    fw = np.zeros(3 * m)
    valid = np.zeros(m, np.int32)
    stats = np.zeros(7 * nb)
    fin = np.zeros(1, np.int32)
    mf = np.zeros(1)
    for k in range(steps):
        f = sc.frame(k)
        R.ref_set_frame(h, *(B.dptr(np.ascontiguousarray(v, dtype=np.float64))
                             for v in (f.p, f.pd, f.pdd, f.q, f.omega, f.alpha)))
        pts, vel, nrm, area = sc.markers(k)
        R.ref_session_step(h, nb, B.i64ptr(sc.offsets), B.dptr(pts.reshape(-1)),
                           B.dptr(vel.reshape(-1)), B.dptr(nrm.reshape(-1)), B.dptr(area),
                           B.dptr(fw), B.iptr(valid), B.dptr(stats), B.iptr(fin), B.dptr(mf))
        assert fin[0] == 1 and mf[0] > -1e-3, k
    n = sc.n_cells
    rho, u, F = np.empty(n), np.empty(3 * n), np.empty(3 * n)
    R.ref_get_macro(h, B.dptr(rho), B.dptr(u))
    R.ref_get_force(h, B.dptr(F))
    R.ref_session_destroy(h)
    return dict(rho=rho, u=u.reshape(-1, 3), F=F.reshape(-1, 3), fw=fw, valid=valid)


def test_c1_1000_steps_vs_reference():
    """BASELINE configs[0] -- 64^3, one rigid sphere, IB on, 1000 steps, the
    CPU-runnable oracle case -- through the reference itself: parity mode
    bit-exact, throughput mode within 1e-5 on rho - 1, u, F and the marker
    forces, stencil sets identical."""
    from oracle import bind as B
    if not B.have_ref():
        pytest.skip("oracle/_ref (the compiled reference) not built")
    sc, out = _run_pair("c1", 1000)
    ref = _run_reference_c1(sc, 1000)
    g64 = out["fp64"]
    for key in ("rho", "u", "F", "fw", "valid"):
        assert np.array_equal(np.asarray(g64[key]).reshape(-1), np.asarray(ref[key]).reshape(-1)), key
    ref["st"] = g64["st"]
    _assert_tol(out["fp32"], ref, "c1 fp32 vs reference after 1000 steps")


def test_force_capture_is_the_consumed_field():
    """The captured fp32 field agrees with the fp64 rebuild of the same step
    (IB band decoded from 2^-40 fixed point, plus the virtual force) to fp32
    rounding, and capture does not change the step's results."""
    from paper_2206_01683_b200.scenes import make_scene
    sc = make_scene("c2")
    res = []
    for cap in (False, True):
        s = _session(sc, "fp32")
        s.set_force_capture(cap)
        for k in range(5):
            s.set_frame(sc.frame(k))
            s.set_markers(sc.offsets, *sc.markers(k))
            s.step()
        rho, u = s.macro()
        res.append((rho, u, s.force(), s.marker_forces()[0]))
        s.close()
    (r0, u0, F_rebuild, fw0), (r1, u1, F_cap, fw1) = res
    assert np.array_equal(r0, r1) and np.array_equal(u0, u1) and np.array_equal(fw0, fw1)
    assert np.abs(F_cap).max() > 0
    assert K.rel_l2(F_cap, F_rebuild) <= 1e-6


def test_skinned_c2_10k_steps_run_to_run_bit_identical():
    """Race evidence for the banded PDL schedule (stamps published by the
    marker grid, acquired by K4 before its first stamp load): two 10,000-step
    runs of the device-skinned c2 step (the bench's coupled path) end in
    bit-identical distributions, marker forces and tau_ext."""
    from paper_2206_01683_b200.scenes import make_scene
    sc = make_scene("c2")
    outs = []
    for _ in range(2):
        s = _session(sc, "fp32")
        s.set_force_capture(False)
        s.set_skin(*sc.skin())
        for k in range(10_000):
            st, tau, _ = s.step_skinned(sc.frame(k), sc.poses(k))
        assert st.stable()
        outs.append((s.get_f(), s.marker_forces()[0], [np.array(t) for t in tau]))
        s.close()
    (f0, m0, t0), (f1, m1, t1) = outs
    assert np.array_equal(f0, f1)
    assert np.array_equal(m0, m1)
    for a, b in zip(t0, t1):
        assert np.array_equal(np.asarray(a), np.asarray(b))
