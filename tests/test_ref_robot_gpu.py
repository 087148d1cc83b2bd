"""GPU: the device robot path against the REFERENCE'S OWN robot code.

The fixtures tests/golden/ref_robot_<design>.npz were produced by the
reference's robot/, empirical/ headers compiled unmodified into oracle/_ref
(tests/golden/make_ref_robot_golden.py), on the reference's own fish
(build_fish_model, model_builder.hpp:104-264) and its own surface samples
(sample_surface, sampling.hpp:164-303).  Here the product runs on exactly
those models and samples:

* fsg_dyn (RobotBatch) -- the robot half of CoupledSession::step
  (session.hpp:167-175; dynamics.hpp:23-289): one step from each reference
  state within rel 1e-12, the 100-step trajectory within rel 1e-10;
* fsg_set_skin / device update_samples (sampling.hpp:307-322) in both
  precisions: markers within rel 1e-13 of the reference's; tau_ext and
  CouplingStats of the session's own marker forces against the reference's
  accumulate_skinned_force loop (session.hpp:127-143) run live on the same
  forces (fp64 1e-13, fp32 1e-5);
* fsg_drag (DragBatch) -- EmpiricalBackend::step (empirical.hpp:74-100):
  tau_ext and stats of each reference step (fp64 rel 1e-12; fp32 rel 1e-9
  plus the 2^-44 fixed-point resolution per sample term) and the coupled
  robot trajectory within rel 1e-10 after 60 steps.
"""
import os

import numpy as np
import pytest

import ref_models as RM
from oracle import bind as B

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _designs():
    from paper_2206_01683_b200._abi import DYN_MAX_LINKS, SKIN_MAX_LINKS
    out = []
    for d in ("koi", "flatfish", "eel"):
        g = np.load(os.path.join(HERE, "golden", f"ref_robot_{d}.npz"))
        if len(g["links"]) <= min(DYN_MAX_LINKS, SKIN_MAX_LINKS):
            out.append(d)
    return out


def _g(design):
    return np.load(os.path.join(HERE, "golden", f"ref_robot_{design}.npz"))


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("design", _designs())
def test_dynamics_vs_reference(design):
    from paper_2206_01683_b200.dynamics import RobotBatch
    g = _g(design)
    robot = RM.robot_from_packed(g["links"], g["bladder"])
    nj, nd = robot.n_joints, robot.n_dofs
    rb = RobotBatch(robot, 2)
    xs = np.concatenate([g["dyn_x0"][None], g["dyn_x"]])
    # one step from each reference state
    worst1 = 0.0
    for k in range(0, 100, 9):
        sts = [RM.unpack_state(xs[k], nj, nd) for _ in range(2)]
        rb.set_states(sts)
        act = np.tile(g["dyn_act"][k], (2, 1))
        tau = np.tile(g["dyn_tau"][k], (2, 1))
        rb.step(act, tau, 1000.0, (0.0, 0.0, -9.81), 0.004, 4)
        for st in rb.states():
            worst1 = max(worst1, _rel(RM.pack_state(st), xs[k + 1]))
    assert worst1 <= 1e-12, worst1
    # the whole trajectory
    rb.set_states([RM.unpack_state(xs[0], nj, nd) for _ in range(2)])
    worst = 0.0
    for k in range(100):
        rb.step(np.tile(g["dyn_act"][k], (2, 1)), np.tile(g["dyn_tau"][k], (2, 1)), 1000.0,
                (0.0, 0.0, -9.81), 0.004, 4)
        worst = max(worst, _rel(RM.pack_state(rb.states()[0]), xs[k + 1]))
    assert worst <= 1e-10, worst
    rb.close()


def _skin_session(g, precision):
    from paper_2206_01683_b200 import CoupledSession, SessionConfig
    m = len(g["areas"])
    s = CoupledSession(SessionConfig(dims=(96, 96, 96), dx=0.01, dt=0.002, rho=1000.0, nu=1e-3,
                                     frame_mode="none", precision=precision, max_markers=m))
    s.set_skin(np.array([0, m], dtype=np.int64), [RM.skeleton_from_packed(g["links"])],
               g["rest_points"], g["rest_normals"], [g["weights"]], g["areas"])
    return s


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("design", _designs())
def test_skinning_and_tau_vs_reference(design, precision):
    g = _g(design)
    s = _skin_session(g, precision)
    live = B.have_ref()
    if live:
        model = RM.RefModel(design)
        S = RM.RefSamples(model, 0.02, 1234)
        assert S.m == len(g["areas"])
    for i in range(len(g["skin_x"])):
        x = g["skin_x"][i].copy()
        x[:3] *= 0.5  # keep the body inside the 0.96 m box
        kc = model.kinematics(x) if live else None
        if not live:
            if i:
                break
            x, kc = g["skin_x"][i], g["skin_kc"][i]
        st, tau, stats = s.step_skinned(None, RM.pose_from_kc(kc)[None])
        pts, vel, nrm = s.markers()
        if live:
            rp, rv, rn = S.update(x)
        else:
            rp, rv, rn = g["skin_pts"][i], g["skin_vel"][i], g["skin_nrm"][i]
        for a, b in ((pts, rp), (vel, rv), (nrm, rn)):
            assert _rel(a, b) <= 1e-13
        if not live:
            continue
        fw, valid, _ = s.marker_forces()
        assert valid.sum() > 0.9 * len(valid) and np.abs(fw).max() > 0
        rtau, rst = S.skinned_tau(x, fw, valid)
        tol = 1e-13 if precision == "fp64" else 1e-5
        assert _rel(tau[0], rtau) <= tol, (i, _rel(tau[0], rtau))
        assert _rel(stats[0], rst[:7]) <= tol
    s.close()


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("design", _designs())
def test_empirical_drag_vs_reference(design, precision):
    from paper_2206_01683_b200 import DragBatch
    from paper_2206_01683_b200.dynamics import RobotBatch
    g = _g(design)
    robot = RM.robot_from_packed(g["links"], g["bladder"])
    robot.bladder.volume = float(g["emp_bladder"][0])
    nj, nd = robot.n_joints, robot.n_dofs
    d = DragBatch(1, k=40.0, precision=precision)
    d.set_skin(0, RM.skeleton_from_packed(g["links"]), g["rest_points"], g["rest_normals"],
               g["weights"], g["areas"])
    # fp32 mode reduces through 2^-44 fixed point: each sample's term is
    # rounded once, so the absolute error is bounded by (terms) * 2^-45
    tol = 1e-12 if precision == "fp64" else 1e-9
    atol = 1e-15 if precision == "fp64" else 4 * len(g["areas"]) * 2.0 ** -45
    for k in range(60):
        d.set_pose(0, RM.pose_from_kc(g["emp_kc"][k]))
        tau, stats = d.step()
        assert np.allclose(tau[0], g["emp_tau"][k], rtol=tol, atol=atol), k
        assert np.allclose(stats[0][3:7], g["emp_stats"][k][3:7], rtol=tol, atol=atol), k
    # and the coupled trajectory: drag on the device feeding the device robot step
    rb = RobotBatch(robot, 1)
    rb.set_states([RM.unpack_state(g["emp_x0"], nj, nd)])
    worst = 0.0
    for k in range(60):
        st = rb.states()[0]
        d.set_pose(0, rb.poses(*RM_rest(robot))[0])
        tau, _ = d.step()
        rb.step(g["emp_act"][k][None], tau[0][None], 1000.0, (0.0, 0.0, -9.81), 0.004, 4)
        worst = max(worst, _rel(RM.pack_state(rb.states()[0]), g["emp_x"][k]))
        assert st is not None
    assert worst <= 1e-10, worst
    rb.close()
    d.close()


def RM_rest(robot):
    from paper_2206_01683_b200.dynamics import rest_pose
    return rest_pose(robot)
