"""GPU: a blown-up step delivers NaN tau_ext, as the reference would.

The throughput reductions of tau_ext / CouplingStats go through 64-bit fixed
point (2^-44) integer atomics; a NaN or out-of-range term used to wrap to a
finite INT64_MIN-scaled value, so a diverged fluid handed the robot step a
finite but wrong tau_ext.  Now such a term sets a per-body flag
and the conversion writes NaN -- the reference propagates the NaN of a
diverged fluid into tau_ext (session.hpp:127-143) and on into the robot
state, where FSG_DYN_NONFINITE catches it.  The flag is cleared with the
sums: the next healthy step is finite again.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _skin_session(sc, E=None):
    from paper_2206_01683_b200 import CoupledSession, EnvBatch, SessionConfig
    cfg = SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                        frame_mode=sc.frame_mode, precision="fp32", max_markers=sc.m)
    if E is None:
        s = CoupledSession(cfg)
        s.set_skin(*sc.skin())
        return s
    b = EnvBatch(cfg, E)
    for s in b.envs:
        s.set_skin(*sc.skin())
    return b


def test_fused_skin_tau_nan_on_nonfinite_fluid():
    from paper_2206_01683_b200.scenes import make_scene
    sc = make_scene("c5")
    s = _skin_session(sc)
    st, tau, stats = s.step_skinned(sc.frame(0), sc.poses(0))
    assert np.isfinite(tau[0]).all() and np.abs(tau[0]).max() > 0
    s.set_f(np.full(19 * sc.n_cells, np.nan))
    st, tau, stats = s.step_skinned(sc.frame(1), sc.poses(1))
    assert not st.stable()
    assert np.isnan(tau[0]).all() and np.isnan(stats[0][3:]).all()
    s.reset_to_rest()
    st, tau, stats = s.step_skinned(sc.frame(2), sc.poses(2))  # flag cleared with the sums
    assert st.stable() and np.isfinite(tau[0]).all()
    s.close()


def test_batch_tau_nan_only_in_the_blown_up_env():
    from paper_2206_01683_b200.scenes import make_scene
    sc = make_scene("c5")
    b = _skin_session(sc, E=2)
    fr = [sc.frame(0), sc.frame(37)]
    po = np.stack([sc.poses(0)[0], sc.poses(37)[0]])
    b.step_skinned(fr, po)
    b.envs[0].set_f(np.full(19 * sc.n_cells, np.nan))
    sts, taus, stats = b.step_skinned(fr, po)
    assert np.isnan(taus[0]).all() and np.isfinite(taus[1]).all()
    assert sts[1].stable() and not sts[0].stable()
    b.envs[0].reset_to_rest()
    sts, taus, stats = b.step_skinned(fr, po)
    assert np.isfinite(taus[0]).all() and np.isfinite(taus[1]).all()
    b.close()


def test_drag_tau_nan_on_nonfinite_pose():
    from paper_2206_01683_b200 import DragBatch
    from paper_2206_01683_b200.scenes import make_scene
    sc = make_scene("c5")
    off, sks, rest, nrest, W, areas = sc.skin()
    d = DragBatch(2, k=40.0, precision="fp32")
    for e in range(2):
        d.set_skin(e, sks[0], rest, nrest, W[0], areas)
    bad = sc.poses(3)[0].copy()
    bad[:] = np.nan
    d.set_pose(0, bad)
    d.set_pose(1, sc.poses(5)[0])
    tau, stats = d.step()
    assert np.isnan(tau[0]).all() and np.isfinite(tau[1]).all()
    d.set_pose(0, sc.poses(3)[0])
    tau, stats = d.step()
    assert np.isfinite(tau[0]).all()
    d.close()
