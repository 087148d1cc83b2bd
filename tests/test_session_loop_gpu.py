"""GPU: the reference's WHOLE CoupledSession::step with the robot on the device.

sim::CoupledSession (session.hpp:29-241) is compiled unmodified into
oracle/_ref (oracle/ref_robot.cpp) and run live on the box's CPU with the
reference's own koi and eel (build_fish_model(koi_design() / eel_design());
the eel's 11 links / 16 dofs exercise the raised caps), its own surface samples
(sample_surface at the lattice spacing) and a SineGait (gait.hpp:12-40).  The
product runs the same session through fsg_batch_step_dynamic (EnvBatch.
step_dynamic): device skinning of the samples, IB coupling + the banded
collide/stream in the followed frame, tau_ext straight into the device robot
step, then the FrameFollower and the integer-cell recentre trigger
(session.hpp:177-195) -- no prescribed frames, no host marker state.

The product's fluid is fp32 (the batch runs the throughput step), so the
comparison is to tolerance: after 300 koi / 200 eel steps (recentre
threshold 0.5 cells so the slow start of the gait already triggers 5 / 9
shifts) the robot state and frame agree with the reference to rel 1e-6
(measured ~5e-9) and tau_ext and f - w to rel-L2 1e-5 (measured 1.3e-7 and
2-4e-7); the distributions only agree if every recentre shift matched.
"""
import math

import numpy as np
import pytest

from oracle import bind as B

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not B.have_ref(), reason="oracle/_ref (the compiled reference) not built")]

W = np.array([1 / 3] + [1 / 18] * 6 + [1 / 36] * 12)


def _gait(links, t):
    """SineGait::actuation defaults (gait.hpp:24-40) on packed reference links."""
    T = 0.5
    r = math.sin(0.5 * math.pi * t / T) if t < T else 1.0
    out, rank = [], 0
    for o in links[1:]:
        if int(o[1]) != 1:
            continue
        ax = o[14:17] / np.linalg.norm(o[14:17])
        if abs(ax[2]) > 0.9:
            out.append(o[35] * (r * 0.6 * math.sin(2 * math.pi * 2.0 * t - rank * 0.8)))
            rank += 1
        else:
            out.append(0.0)
    return np.array(out)


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("design,frame_mode,steps", [("koi", "translation_yaw", 300),
                                                     ("koi", "none", 120),
                                                     ("eel", "translation_yaw", 200)])
def test_coupled_session_loop_vs_reference(design, frame_mode, steps):
    import ref_models as RM
    from paper_2206_01683_b200 import EnvBatch, SessionConfig
    from paper_2206_01683_b200.dynamics import RobotBatch, rest_pose
    # the eel (0.6 m, 11 links, 16 dofs) in a longer box
    dims = (64, 32, 32) if design == "koi" else (96, 32, 32)
    dx, dt, rho, nu = 0.01, 0.004, 1000.0, 0.00089
    fm = {"none": 0, "translation_yaw": 2}[frame_mode]
    model = RM.RefModel(design)
    ref = RM.SessionRef(dims, dx, dt, rho, nu, kernel=0, wall=0, frame_mode=fm, frame_tc=0.2,
                        recenter_cells=0.5, gravity=(0.0, 0.0, -9.81), substeps=4,
                        marker_spacing=0.0)
    ref.add_robot(model, pos=(0.0, 0.0, 0.0), yaw=0.0, seed=1234)
    x0, _, _, bladder = ref.robot(0)
    P, N, A, Wt = model.samples(dx, 1234)  # add_robot's sample_surface(mesh, dx, seed)
    m = len(A)
    robot = model.robot()
    robot.bladder.volume = bladder  # apply_start: neutral trim in the session's fluid
    cfg = SessionConfig(dims=dims, dx=dx, dt=dt, rho=rho, nu=nu, frame_mode=frame_mode,
                        precision="fp32", max_markers=m)
    b = EnvBatch(cfg, 1)
    b.envs[0].set_skin(np.array([0, m], dtype=np.int64), [model.skeleton()], P, N, [Wt], A)
    rb = RobotBatch(robot, 1)
    rb.set_rest(*rest_pose(robot))
    rb.set_states([model.unpack(x0)])
    if frame_mode != "none":
        b.set_follow(0.2, 0.5)
        b.center_frames(rb)
        assert np.allclose(b.envs[0].frame_state().packed()[:3], ref.frame()[:3])
    n_shift = 0
    for k in range(steps):
        act = _gait(model.links, k * dt)
        ref.set_actuation(0, act)
        ok, oob = ref.step()
        assert ok and oob == 0, k
        st, fl, packed = b.step_dynamic(rb, act[None])
        assert st[0].stable() and fl[0] == 0, k
        if frame_mode != "none":
            sh = b.last_shifts()[0]
            n_shift += int(np.abs(sh).sum() > 0)
    xr, tr, sr, _ = ref.robot(0)
    xg = RM.pack_state(rb.states()[0])
    assert _rel(xg, xr) <= 1e-6, _rel(xg, xr)
    assert np.abs(xr[:3]).max() > 0.5 * dx  # the koi actually swam
    tau_g, stats_g = b.envs[0].body_wrench()
    assert _rel(tau_g[0], tr) <= 1e-5, _rel(tau_g[0], tr)
    if frame_mode != "none":
        assert n_shift >= 1  # the trigger fired (and the fields below only agree if it matched)
        fg = b.envs[0].frame_state().packed()
        assert _rel(fg[:3], ref.frame()[:3]) <= 1e-6
        assert _rel(fg[9:13], ref.frame()[9:13]) <= 1e-6
    n = int(np.prod(dims))
    fr = ref.get_f().reshape(19, n) - W[:, None]
    fgd = b.envs[0].get_f().reshape(19, n) - W[:, None]
    assert _rel(fgd, fr) <= 1e-5, _rel(fgd, fr)
    print(f"{design} {frame_mode} {steps} steps: state rel {_rel(xg, xr):.2e}, tau_ext rel "
          f"{_rel(tau_g[0], tr):.2e}, f - w rel-L2 {_rel(fgd, fr):.2e}, recentres {n_shift}")
    b.close()
    rb.close()
