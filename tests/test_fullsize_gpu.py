"""Parity at the BASELINE configs' full sizes, where the CPU oracle is too
slow to run: the fp32 throughput mode against the fp64 parity mode (itself
bit-identical to the reference, test_parity_gpu.py) on the c2 and c3 scenes,
and size-independent invariants on the 512^3 grid (c4): exact mass
conservation in a periodic box and Guo forcing's exact momentum injection
(solver.hpp:129-154: the bare momentum grows by F per cell per step)."""
import numpy as np
import pytest

import cases as K
from paper_2206_01683_b200 import CoupledSession, FrameState, SessionConfig
from paper_2206_01683_b200.scenes import make_scene

pytestmark = pytest.mark.gpu
TOL32 = 1e-5


@pytest.mark.parametrize("name,steps", [("c2", 20), ("c3", 8)])
def test_scene_fp32_vs_fp64_parity_mode(name, steps):
    sc = make_scene(name)
    out = {}
    for prec in ("fp64", "fp32"):
        s = CoupledSession(SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                                         frame_mode=sc.frame_mode, precision=prec, max_markers=sc.m))
        for k in range(steps):
            s.set_frame(sc.frame(k))
            s.set_markers(sc.offsets, *sc.markers(k))
            assert s.step().stable()
        fw, valid, stats = s.marker_forces()
        rho, u = s.macro()
        out[prec] = dict(u=u, rho=rho, fw=fw, valid=valid, stats=stats, st=s.stencils())
        s.close()
    a, b = out["fp32"], out["fp64"]
    assert np.array_equal(a["st"], b["st"]), "stencil index sets differ"
    assert np.array_equal(a["valid"], b["valid"])
    assert K.rel_l2(a["u"], b["u"]) <= TOL32
    assert K.rel_l2(a["rho"] - 1.0, b["rho"] - 1.0) <= TOL32
    assert K.rel_l2(a["fw"], b["fw"]) <= TOL32
    assert K.rel_l2(a["stats"], b["stats"]) <= TOL32


def test_c4_512cubed_mass_and_momentum_invariants():
    dims, dx, dt = (512, 512, 512), 0.01, 0.004
    n = dims[0] * dims[1] * dims[2]
    pdd = np.array([0.1, -0.05, 0.02])
    s = CoupledSession(SessionConfig(dims=dims, dx=dx, dt=dt, boundary="periodic",
                                     frame_mode="translation", precision="fp32", max_markers=1))
    s.reset_to_rest()
    m0 = s.total_mass()
    s.set_frame(FrameState(pdd=pdd))
    steps = 3
    for _ in range(steps):
        assert s.step().stable()
    # uniform force in a periodic box: rho stays 1, so F = acc * (-pdd) per cell
    F = (dt * dt / dx) * (-pdd)
    mom = s.total_momentum()
    assert abs(s.total_mass() - m0) <= 1e-6 * m0
    assert np.abs(mom - steps * n * F).max() <= 1e-5 * np.abs(steps * n * F).max()
    s.close()
