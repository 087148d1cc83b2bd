"""CPU tests of the oracle (test infrastructure): it must agree bit-for-bit
with the reference's own code (golden fixtures made by oracle/_ref, and the
live _ref build when present), and satisfy the reference's own known-answer
tests (test_lattice.cpp, test_ib.cpp, test_frame.cpp) re-expressed here."""
import math
import os

import numpy as np
import pytest

import cases as K
from oracle import bind as B

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    z = np.load(os.path.join(GOLD, name + ".npz"))
    return {k[4:]: z[k] for k in z.files if k.startswith("out_")}


O = B.oracle()


# ------------------------------------------------------- golden vectors -----
@pytest.mark.parametrize("mk", [K.case_lbm_open, K.case_lbm_periodic])
def test_oracle_lbm_matches_reference_golden(mk):
    c = mk()
    g = gold(c["name"])
    r = K.run_oracle_lbm(c)
    for key in ("f", "min_f", "finite", "rho", "u", "momentum"):
        assert np.array_equal(np.asarray(r[key]), g[key]), key
    assert r["mass"] == g["mass"] and r["nonpos"] == g["nonpos"]


@pytest.mark.parametrize("mk", [K.case_session_frame, K.case_session_roma3])
def test_oracle_session_matches_reference_golden(mk):
    c = mk()
    g = gold(c["name"])
    r = K.run_oracle_session(c)
    for key in ("f", "rho", "u", "F", "fw", "valid", "stats", "min_f", "finite", "nonpos", "oob",
                "frame_p_rc"):
        assert np.array_equal(np.asarray(r[key]), g[key]), key


def test_oracle_ib_primitives_match_reference_golden():
    z = np.load(os.path.join(GOLD, "ib_primitives.npz"))
    for k in (0, 1):
        phi = np.array([O.orc_phi(k, float(r)) for r in z["rs"]])
        assert np.array_equal(phi, z["out_phi"][k])
        for i, x in enumerate(z["xs"]):
            lo = np.zeros(1, np.int32)
            hi = np.zeros(1, np.int32)
            O.orc_range(k, float(x), B.iptr(lo), B.iptr(hi))
            assert (lo[0], hi[0]) == tuple(z["out_range"][k, i])


@pytest.mark.skipif(not B.have_ref(), reason="oracle/_ref not built (needs /root/reference)")
def test_rng_restatement_matches_reference():
    R = B.ref()
    out = np.zeros(64)
    R.ref_rng_uniform(7, 64, B.dptr(out))
    r = B.Rng(7)
    assert np.array_equal(out, r.uniforms(64))


@pytest.mark.skipif(not B.have_ref(), reason="oracle/_ref not built (needs /root/reference)")
def test_oracle_matches_live_reference_random_session():
    """Fresh random case (not a fixture) through both the compiled reference and the oracle."""
    c = K.case_session_frame()
    rng = np.random.default_rng(123)
    n = int(np.prod(c["dims"]))
    c.update(rho0=1.0 + 0.01 * (rng.random(n) - 0.5), u0=0.02 * (rng.random(3 * n) - 0.5),
             script=[("step", 0), ("step", 1), ("recenter", (-1, 2, 0)), ("step", 2)])
    a = K.run_ref_session(c)
    b = K.run_oracle_session(c)
    for key in ("f", "rho", "u", "F", "fw", "valid", "stats", "min_f", "frame_p_rc"):
        assert np.array_equal(np.asarray(a[key]), np.asarray(b[key])), key


@pytest.mark.skipif(not B.have_ref(), reason="oracle/_ref not built (needs /root/reference)")
def test_oracle_virtual_force_and_direct_forcing_match_reference():
    R = B.ref()
    rng = np.random.default_rng(4)
    for _ in range(50):
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        pdd, om, al, x, u = (rng.normal(size=3) for _ in range(5))
        a = np.zeros(3)
        R.ref_virtual_force(*(B.dptr(B.d3(v)) for v in (q, pdd, om, al, x, u)), B.dptr(a))
        fs = B.FrameState.make(pdd=pdd, q=q, omega=om, alpha=al)
        fc = B.FrameConsts()
        O.orc_frame_consts_of(fs, fc)
        b = np.zeros(3)
        O.orc_virtual_force(fc, B.dptr(B.d3(x)), B.dptr(B.d3(u)), B.dptr(b))
        assert np.array_equal(a, b)
        ub, uf, nn = (rng.normal(size=3) for _ in range(3))
        for wall in (0, 1):
            f1 = np.zeros(3)
            f2 = np.zeros(3)
            R.ref_direct_forcing(B.dptr(B.d3(ub)), B.dptr(B.d3(uf)), B.dptr(B.d3(nn)), 1000.0, 1e-4,
                                 0.02, 0.004, wall, B.dptr(f1))
            O.orc_direct_forcing(B.dptr(B.d3(ub)), B.dptr(B.d3(uf)), B.dptr(B.d3(nn)), 1000.0, 1e-4,
                                 0.02, 0.004, wall, B.dptr(f2))
            assert np.array_equal(f1, f2)


# ----------------------------- reference KATs re-expressed on the oracle ----
W = K.W


def test_equilibrium_rest_weights_and_linearity():  # test_lattice.cpp:35-48
    for i in range(19):
        assert O.orc_equilibrium_dir(i, 1.0, B.dptr(np.zeros(3))) == pytest.approx(W[i], abs=1e-15)
        assert O.orc_equilibrium_dir(i, 2.0, B.dptr(np.zeros(3))) == pytest.approx(2 * W[i], abs=1e-15)


def test_opposite_directions_negate():  # test_lattice.cpp:67-74
    for i in range(1, 19):
        j = i + 1 if i % 2 == 1 else i - 1
        assert (K.EX[i], K.EY[i], K.EZ[i]) == (-K.EX[j], -K.EY[j], -K.EZ[j])


def _periodic_run(d, tau, f, F, steps):
    dims = B.dims_arr(d)
    fa = f.copy()
    fb = np.empty_like(fa)
    fin = np.zeros(1, np.int32)
    mf = np.zeros(1)
    for _ in range(steps):
        O.orc_collide_and_stream(B.iptr(dims), 1, tau, B.dptr(fa), B.dptr(fb), B.dptr(F), B.iptr(fin),
                                 B.dptr(mf))
        fa, fb = fb, fa
    return fa


def test_mass_momentum_conserved_periodic():  # test_lattice.cpp:164-187
    c = K.case_lbm_periodic()
    d = c["dims"]
    n = int(np.prod(d))
    f = _periodic_run(d, 0.8, c["f0"], np.zeros(3 * n), 300)
    dims = B.dims_arr(d)
    m0, m1 = O.orc_total_mass(B.iptr(dims), B.dptr(c["f0"])), O.orc_total_mass(B.iptr(dims), B.dptr(f))
    p0, p1 = np.zeros(3), np.zeros(3)
    O.orc_total_momentum(B.iptr(dims), B.dptr(c["f0"]), B.dptr(p0))
    O.orc_total_momentum(B.iptr(dims), B.dptr(f), B.dptr(p1))
    assert abs(m1 - m0) / m0 < 1e-12
    assert np.linalg.norm(p1 - p0) < 1e-10


def test_guo_forcing_injects_momentum():  # test_lattice.cpp:189-202
    d = (8, 8, 8)
    n = 512
    f0 = np.repeat(W, n)
    F = np.tile([1e-4, 0.0, 0.0], n)
    f = _periodic_run(d, 0.8, f0, F, 50)
    rho = np.empty(n)
    u = np.empty(3 * n)
    O.orc_macroscopic(B.iptr(B.dims_arr(d)), B.dptr(f), B.dptr(F), B.dptr(rho), B.dptr(u))
    assert np.allclose(u[0::3], 50.5 * 1e-4, rtol=1e-10)


def test_uniform_equilibrium_is_fixed_point_open_and_periodic():  # test_lattice.cpp:115-133
    d = (12, 10, 9)
    n = int(np.prod(d))
    u0 = np.tile([0.04, 0.01, -0.02], n)
    f0 = np.empty(19 * n)
    O.orc_initialize(B.iptr(B.dims_arr(d)), B.dptr(np.ones(n)), B.dptr(u0), B.dptr(f0))
    for periodic in (0, 1):
        fa = f0.copy()
        fb = np.empty_like(fa)
        fin = np.zeros(1, np.int32)
        mf = np.zeros(1)
        for _ in range(5):
            O.orc_collide_and_stream(B.iptr(B.dims_arr(d)), periodic, 0.9, B.dptr(fa), B.dptr(fb),
                                     B.dptr(np.zeros(3 * n)), B.iptr(fin), B.dptr(mf))
            fa, fb = fb, fa
            assert fin[0] == 1 and mf[0] > -1e-3
        assert np.abs(fa - f0).max() < 1e-14


def test_taylor_green_decay_rate():  # test_lattice.cpp:204-234
    N, tau, u0 = 32, 0.8, 0.02
    nu = (tau - 0.5) / 3
    a = 2 * math.pi / N
    z, y, x = np.meshgrid(np.arange(N), np.arange(N), np.arange(N), indexing="ij")
    x, y = x.reshape(-1), y.reshape(-1)
    rho = 1.0 + 3.0 * (-u0 * u0 / 4.0 * (np.cos(2 * a * x) + np.cos(2 * a * y)))
    u = np.stack([u0 * np.cos(a * x) * np.sin(a * y), -u0 * np.sin(a * x) * np.cos(a * y),
                  np.zeros_like(x, dtype=float)], axis=1).reshape(-1)
    d = (N, N, N)
    dims = B.dims_arr(d)
    n = N ** 3
    f = np.empty(19 * n)
    O.orc_initialize(B.iptr(dims), B.dptr(np.ascontiguousarray(rho)), B.dptr(np.ascontiguousarray(u)), B.dptr(f))
    rate = 4.0 * nu * a * a
    t1 = 20
    t2 = t1 + int(1.0 / rate)

    def ke(ff):
        r = np.empty(n)
        uu = np.empty(3 * n)
        O.orc_macroscopic(B.iptr(dims), B.dptr(ff), None, B.dptr(r), B.dptr(uu))
        return float((0.5 * r * (uu.reshape(-1, 3) ** 2).sum(1)).sum())

    F = np.zeros(3 * n)
    fa, fb = f, np.empty_like(f)
    fin = np.zeros(1, np.int32)
    mf = np.zeros(1)
    for s in range(t2 + 1):
        if s == t1:
            e1 = ke(fa)
        O.orc_collide_and_stream(B.iptr(dims), 1, tau, B.dptr(fa), B.dptr(fb), B.dptr(F), B.iptr(fin),
                                 B.dptr(mf))
        fa, fb = fb, fa
    e2 = ke(fa)
    assert abs(math.log(e1 / e2) / (t2 + 1 - t1) / rate - 1.0) < 0.03


def test_ib_partition_of_unity_and_first_moment():  # test_ib.cpp:30-45
    r = B.Rng(2)
    for k in (0, 1):
        for _ in range(200):
            x = r.uniform(-0.5, 0.5)
            s = sum(O.orc_phi(k, x - j) for j in range(-4, 5))
            m1 = sum(j * O.orc_phi(k, x - j) for j in range(-4, 5))
            assert abs(s - 1) < 1e-6 and abs(m1 - x) < 1e-6


def test_interp_spread_adjoint():  # test_ib.cpp:136-160
    rng = np.random.default_rng(11)
    d = (12, 14, 13)
    dims = B.dims_arr(d)
    n = int(np.prod(d))
    for trial in range(30):
        k = trial % 2
        u = rng.normal(size=3 * n)
        F = np.zeros(3 * n)
        rhs = 0.0
        for _ in range(1 + trial % 8):
            x = np.array([rng.uniform(2.5, 9.5), rng.uniform(2.5, 11.0), rng.uniform(2.5, 10.0)])
            f = rng.normal(size=3)
            O.orc_spread(k, B.iptr(dims), B.dptr(F), B.dptr(x), B.dptr(f))
            ui = np.zeros(3)
            O.orc_interpolate(k, B.iptr(dims), B.dptr(u), B.dptr(x), B.dptr(ui))
            rhs += f @ ui
        assert abs(F @ u - rhs) <= 1e-10 * max(1.0, abs(rhs))


def test_marker_bounds_margin():  # test_ib.cpp:251-260
    d = B.dims_arr((16, 16, 16))
    ok = lambda k, x: O.orc_marker_in_bounds(k, B.iptr(d), B.dptr(B.d3(x)))
    assert ok(0, (8, 8, 8)) and ok(0, (2.0, 8, 8))
    assert not ok(0, (1.9, 8, 8)) and not ok(0, (8, 13.1, 8))
    assert ok(1, (1.6, 8, 8))


def test_virtual_force_kats():  # test_frame.cpp:14-54
    fc = B.FrameConsts()
    O.orc_frame_consts_of(B.FrameState.make(pd=(1.0, -0.5, 0.2)), fc)
    a = np.zeros(3)
    O.orc_virtual_force(fc, B.dptr(B.d3((0.3, 0.1, -2))), B.dptr(B.d3((1, 2, 3))), B.dptr(a))
    assert np.linalg.norm(a) == 0.0
    w, R = 1.7, 0.8
    for yaw in (0.0, 1.2):
        O.orc_frame_consts_of(B.FrameState.make(omega=(0, 0, w), q=(math.cos(yaw / 2), 0, 0,
                                                                      math.sin(yaw / 2))), fc)
        O.orc_virtual_force(fc, B.dptr(B.d3((R, 0, 0))), B.dptr(np.zeros(3)), B.dptr(a))
        assert np.linalg.norm(a - [w * w * R, 0, 0]) < 1e-13
