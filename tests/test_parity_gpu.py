"""GPU parity: the CUDA product (through the C ABI) vs the reference.

* FP64 (parity mode) must be BIT-IDENTICAL to the golden fixtures, which
  were produced by the reference's own headers (tests/golden/make_golden.py),
  and to the C oracle on larger seeded cases.
* FP32 (throughput mode) must reproduce the integer stencil sets and marker
  validity exactly and the fields within the stated tolerances:
      rel-L2(u) <= 1e-5, rel-L2(rho - 1) <= 1e-5, rel-L2(F) <= 1e-5,
      rel-L2(marker force) <= 1e-5, rel-L2(f - w) <= 1e-5
  (north_star: "fp32 density, velocity and body-force fields within a
  stated relative-L2 tolerance (e.g. <=1e-5 after N steps)").
"""
import os

import numpy as np
import pytest

import cases as K

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL32 = 1e-5


def gold(name):
    z = np.load(os.path.join(GOLD, name + ".npz"))
    return {k[4:]: z[k] for k in z.files if k.startswith("out_")}


def dev(f, n):
    return f.reshape(19, n) - K.W[:, None]


@pytest.mark.parametrize("mk", [K.case_lbm_open, K.case_lbm_periodic])
def test_collide_and_stream_fp64_bit_exact(mk):
    c = mk()
    g = gold(c["name"])
    r = K.run_gpu_lbm(c, "fp64")
    assert np.array_equal(r["f"], g["f"]), "distributions differ from the reference"
    assert np.array_equal(r["min_f"], g["min_f"])
    assert np.array_equal(r["finite"], g["finite"])
    assert np.array_equal(r["rho"], g["rho"]) and np.array_equal(r["u"], g["u"])
    assert r["nonpos"] == g["nonpos"]
    # reductions: deterministic tree order vs the reference's serial order
    assert abs(r["mass"] - g["mass"]) <= 1e-13 * abs(g["mass"])
    # (momentum: cancellation over 19 n terms of O(w); scale by the mass)
    assert np.abs(r["momentum"] - g["momentum"]).max() <= 1e-13 * abs(g["mass"])


@pytest.mark.parametrize("mk", [K.case_lbm_open, K.case_lbm_periodic])
def test_collide_and_stream_fp32_tolerance(mk):
    c = mk()
    g = gold(c["name"])
    r = K.run_gpu_lbm(c, "fp32")
    n = int(np.prod(c["dims"]))
    assert K.rel_l2(dev(r["f"], n), dev(g["f"], n)) <= TOL32
    assert K.rel_l2(r["u"], g["u"]) <= TOL32
    assert K.rel_l2(r["rho"] - 1.0, g["rho"] - 1.0) <= TOL32
    assert np.all(r["finite"] == 1)
    assert np.allclose(r["min_f"], g["min_f"], rtol=1e-5, atol=1e-7)


@pytest.mark.parametrize("mk", [K.case_session_frame, K.case_session_roma3])
def test_session_step_fp64_bit_exact(mk):
    c = mk()
    g = gold(c["name"])
    r = K.run_gpu_session(c, "fp64")
    assert np.array_equal(r["stencils"], g["stencils"]), "stencil index sets differ"
    assert np.array_equal(r["valid"], g["valid"])
    assert np.array_equal(r["oob"], g["oob"])
    assert np.array_equal(r["fw"], g["fw"]), "marker forces differ"
    assert np.array_equal(r["stats"], g["stats"])
    assert np.array_equal(r["rho"], g["rho"]) and np.array_equal(r["u"], g["u"])
    assert np.array_equal(r["F"], g["F"]), "body force field differs"
    assert np.array_equal(r["f"], g["f"]), "distributions differ"
    assert np.array_equal(r["min_f"], g["min_f"])
    assert np.array_equal(r["finite"], g["finite"])
    assert np.array_equal(r["nonpos"], g["nonpos"])
    assert np.array_equal(r["frame_p_rc"], g["frame_p_rc"])


@pytest.mark.parametrize("mk", [K.case_session_frame, K.case_session_roma3])
def test_session_step_fp32_tolerance(mk):
    c = mk()
    g = gold(c["name"])
    r = K.run_gpu_session(c, "fp32")
    n = int(np.prod(c["dims"]))
    assert np.array_equal(r["stencils"], g["stencils"]), "stencil index sets differ"
    assert np.array_equal(r["valid"], g["valid"])
    assert np.array_equal(r["oob"], g["oob"])
    assert K.rel_l2(r["fw"], g["fw"]) <= TOL32
    assert K.rel_l2(r["u"], g["u"]) <= TOL32
    assert K.rel_l2(r["rho"] - 1.0, g["rho"] - 1.0) <= TOL32
    assert K.rel_l2(r["F"], g["F"]) <= TOL32
    assert K.rel_l2(dev(r["f"], n), dev(g["f"], n)) <= TOL32


def test_recenter_fp64_bit_exact():
    c = K.case_recenter()
    g = gold("recenter")
    from paper_2206_01683_b200 import CoupledSession
    s = CoupledSession(K._gpu_cfg(dict(c, frame_mode=2), "fp64"))
    s.set_f(c["f0"])
    s.set_frame(K._fs_to_product(K.frame_at(3, c["units"]["dt"])))
    for j, sh in enumerate(c["shifts"]):
        s.recenter(sh)
        assert np.array_equal(s.get_f(), g[f"f{j}"])
        assert np.array_equal(s.frame_state().p, g[f"p{j}"])
    s.close()


def test_session_fp64_matches_oracle_larger_case():
    """A larger seeded coupled run (48x40x36, 12 steps + recenter) against the C oracle."""
    c = K.case_session_frame()
    d = (48, 40, 36)
    n = int(np.prod(d))
    r = np.random.default_rng(5)
    c.update(dims=d, rho0=1.0 + 0.01 * (r.random(n) - 0.5), u0=0.01 * (r.random(3 * n) - 0.5))
    pts0, nrm, area = K.fib_sphere(0.09, 1000, np.array([0.01, 0.0, -0.004]))
    c.update(pts0=pts0, nrm=nrm, area=area, offsets=np.array([0, 1000], dtype=np.int64),
             script=[("step", k) for k in range(6)] + [("recenter", (-2, 1, 0))] +
             [("step", k) for k in range(6, 12)])
    o = K.run_oracle_session(c)
    g = K.run_gpu_session(c, "fp64")
    for key in ("f", "rho", "u", "F", "fw", "valid", "min_f", "finite", "nonpos", "oob"):
        assert np.array_equal(np.asarray(g[key]), np.asarray(o[key])), key


def _larger_case(script, jumps=None):
    c = K.case_session_frame()
    d = (48, 40, 36)
    n = int(np.prod(d))
    r = np.random.default_rng(5)
    c.update(dims=d, rho0=1.0 + 0.01 * (r.random(n) - 0.5), u0=0.01 * (r.random(3 * n) - 0.5))
    pts0, nrm, area = K.fib_sphere(0.09, 1000, np.array([0.01, 0.0, -0.004]))
    c.update(pts0=pts0, nrm=nrm, area=area, offsets=np.array([0, 1000], dtype=np.int64),
             script=script, jumps=jumps or {})
    return c


def test_session_fp32_band_misses_match_oracle():
    """Throughput path when the IB band moves unpredictably: the body jumps by
    several cells between steps (and the domain is recentred), so the tiles
    its stencils touch change wholesale from one step to the next.  The fp32
    session must still match the oracle within tolerance every time."""
    jumps = {3: (0.031, 0.0, 0.0), 4: (0.031, -0.022, 0.0), 5: (-0.02, 0.0, 0.027),
             8: (0.0, 0.05, 0.0)}
    c = _larger_case([("step", k) for k in range(6)] + [("recenter", (-2, 1, 0))] +
                     [("step", k) for k in range(6, 10)], jumps)
    o = K.run_oracle_session(c)
    g = K.run_gpu_session(c, "fp32")
    n = int(np.prod(c["dims"]))
    assert np.array_equal(g["valid"], o["valid"]) and np.array_equal(g["oob"], o["oob"])
    assert K.rel_l2(g["fw"], o["fw"]) <= TOL32
    assert K.rel_l2(g["u"], o["u"]) <= TOL32
    assert K.rel_l2(g["rho"] - 1.0, o["rho"] - 1.0) <= TOL32
    assert K.rel_l2(g["F"], o["F"]) <= TOL32
    assert K.rel_l2(dev(g["f"], n), dev(o["f"], n)) <= TOL32


def test_session_fp32_run_to_run_bit_identical():
    """Fixed-point spread + one writer per cell: two identical fp32 runs give
    bit-identical distributions, forces and marker forces."""
    c = _larger_case([("step", k) for k in range(8)])
    a = K.run_gpu_session(c, "fp32")
    b = K.run_gpu_session(c, "fp32")
    for key in ("f", "F", "fw", "min_f"):
        assert np.array_equal(a[key], b[key]), key


def test_c1_scene_fp32_vs_fp64_parity_mode():
    """BASELINE config c1 at full size (64^3, ~2000 markers on a sphere):
    30 coupled steps in throughput mode vs parity mode (fp64, bit-exact to the
    reference by the tests above) on identical inputs."""
    from paper_2206_01683_b200 import CoupledSession, SessionConfig
    from paper_2206_01683_b200.scenes import make_scene
    sc = make_scene("c1")
    out = {}
    for prec in ("fp64", "fp32"):
        s = CoupledSession(SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                                         frame_mode=sc.frame_mode, precision=prec,
                                         max_markers=sc.m))
        for k in range(30):
            s.set_frame(sc.frame(k))
            s.set_markers(sc.offsets, *sc.markers(k))
            st = s.step()
            assert st.stable()
        fw, valid, _ = s.marker_forces()
        rho, u = s.macro()
        out[prec] = dict(u=u, rho=rho, fw=fw, valid=valid, st=s.stencils())
        s.close()
    a, b = out["fp32"], out["fp64"]
    assert np.array_equal(a["st"], b["st"]) and np.array_equal(a["valid"], b["valid"])
    assert K.rel_l2(a["u"], b["u"]) <= TOL32
    assert K.rel_l2(a["rho"] - 1.0, b["rho"] - 1.0) <= TOL32
    assert K.rel_l2(a["fw"], b["fw"]) <= TOL32
