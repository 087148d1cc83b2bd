"""GPU: the synchronous step's status path.

fsg_step (CoupledSession.step) has its status written into pinned host
memory by a one-warp programmatic dependent of K4 (k_step_end); the
asynchronous step leaves it in the device scratch and fsg_last_status copies
it.  Both must report the same StepStatus for the same step -- min_f bit for
bit, the finite flag, the non-positive-density count and the out-of-bounds
marker count -- through healthy steps, markers outside the box and a
blown-up state, and a batched step in between must not leave a stale
published status behind.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _pair(sc):
    from paper_2206_01683_b200 import CoupledSession, SessionConfig
    cfg = SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                        frame_mode=sc.frame_mode, precision="fp32", max_markers=sc.m)
    out = []
    for _ in range(2):
        s = CoupledSession(cfg)
        s.set_skin(*sc.skin())
        out.append(s)
    return out


def _same(a, b):
    assert a.finite == b.finite
    assert a.n_nonpositive_rho == b.n_nonpositive_rho
    assert a.out_of_bounds_markers == b.out_of_bounds_markers
    assert (np.isnan(a.min_f) and np.isnan(b.min_f)) or a.min_f == b.min_f


def test_sync_status_equals_async_status():
    from paper_2206_01683_b200.scenes import make_scene
    sc = make_scene("c2")
    sync, asy = _pair(sc)
    for k in range(6):
        for s in (sync, asy):
            s.set_frame(sc.frame(k))
            s.set_pose(sc.poses(k))
        a = sync.step()
        asy.step_async()
        b = asy.last_status()
        _same(a, b)
        assert a.stable()
        _same(sync.last_status(), a)  # re-reading the published status
    # a blown-up state: non-finite populations reach the status both ways
    for s in (sync, asy):
        s.set_f(np.full(19 * sc.n_cells, np.nan))
        s.set_frame(sc.frame(7))
        s.set_pose(sc.poses(7))
    a = sync.step()
    asy.step_async()
    b = asy.last_status()
    _same(a, b)
    assert not a.finite and not a.stable()
    sync.close()
    asy.close()


def test_async_step_after_sync_step_reports_its_own_status():
    """A published status must not shadow a later asynchronous step's."""
    from paper_2206_01683_b200.scenes import make_scene
    sc = make_scene("c2")
    s, ref = _pair(sc)
    for k in range(2):  # sync, sync: both parities published once
        for x in (s, ref):
            x.set_frame(sc.frame(k))
            x.set_pose(sc.poses(k))
        s.step()
        ref.step()
    for x in (s, ref):
        x.set_f(np.full(19 * sc.n_cells, np.nan))
        x.set_frame(sc.frame(2))
        x.set_pose(sc.poses(2))
    s.step_async()  # this step's status lives in the device scratch only
    ref.step()
    _same(s.last_status(), ref.last_status())
    assert not s.last_status().finite
    s.close()
    ref.close()
