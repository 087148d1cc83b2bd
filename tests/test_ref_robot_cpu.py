"""CPU: the robot-side C restatements pinned to the REFERENCE'S OWN CODE.

oracle/_ref/libfishref.so now also compiles the reference's robot/,
empirical/ and sim/session headers unmodified (oracle/ref_robot.cpp against
the extended Eigen stand-in), so the restatements the GPU tests compare
against (oracle/fsg_dyn_oracle.c, the skinning and drag parts of
oracle/fsg_oracle.c) are checked here against the reference functions they
restate, on the reference's own fish (build_fish_model(koi_design()),
flatfish_design(); model_builder.hpp:104-264) and its own surface samples
(sample_surface, sampling.hpp:164-303):

* robot step (session.hpp:167-175: buoyancy_gravity_forces + integrate with
  4 substeps; dynamics.hpp:23-289) over 300 gait-driven steps: rel <= 1e-12;
* mass_matrix / bias_forces (dynamics.hpp:66-154): rel <= 1e-13;
* update_samples (sampling.hpp:307-322) and the tau_ext / CouplingStats loop
  (session.hpp:127-143, skinning.hpp:147-156): rel <= 1e-13;
* EmpiricalBackend::step (empirical.hpp:74-100), 100 steps: rel <= 1e-12;
* Skeleton::validate messages (skeleton.hpp:96-120).

The stand-in fixes the last-ulp order of Eigen's reductions (LLT, products),
so agreement is to rounding, not bitwise.
"""
import math

import numpy as np
import pytest

from oracle import bind as B

pytestmark = pytest.mark.skipif(not B.have_ref(), reason="oracle/_ref not built")

DESIGNS = ["koi", "flatfish", "eel"]


def _gait(robot, t):
    """SineGait (gait.hpp:12-40) defaults, ramp included."""
    T = 0.5
    r = math.sin(0.5 * math.pi * t / T) if t < T else 1.0
    out, rank = [], 0
    for l in robot.links[1:]:
        if l.joint != 1:
            continue
        ax = np.asarray(l.axis) / np.linalg.norm(l.axis)
        if abs(ax[2]) > 0.9:
            out.append(l.torque_limit * r * 0.6 * math.sin(2 * math.pi * 2.0 * t - rank * 0.8))
            rank += 1
        else:
            out.append(0.0)
    return np.array(out)


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module", params=DESIGNS)
def model(request):
    import ref_models as RM
    return RM.RefModel(request.param)


def test_reference_models_load(model):
    r = model.robot()
    assert r.n_links == model.n_links and r.n_dofs == model.n_dofs
    assert model.floating == 1
    assert abs(r.total_mass() - sum(l.mass for l in r.links)) < 1e-15
    P, N, A, W = model.samples(0.02)
    assert len(A) > 100
    assert np.allclose(W.sum(1), 1.0, atol=1e-12)
    assert (W != 0).sum(1).max() <= 4  # FSG_SKIN_MAX_WEIGHTS


def test_robot_step_restatement_vs_reference(model):
    from paper_2206_01683_b200 import dynamics as D
    r = model.robot()
    O = B.DynOracle(r)
    st = D.JointState.zero(r)
    x = model.zero_state()
    st.base_pos[:] = x[:3] = (0.1, -0.02, 0.05)
    worst = 0.0
    for k in range(300):
        act = _gait(r, k * 0.004)
        tau = 0.02 * np.sin(np.arange(model.n_dofs) * 0.7 + 0.1 * k)
        O.robot_step(st, act, tau, 1000.0, (0.0, 0.0, -9.81), 0.004, 4)
        assert model.step(x, act, tau) == 0
        worst = max(worst, _rel(np.concatenate([st.base_pos, st.base_quat, st.q, st.v]), x))
    assert worst <= 1e-12, worst
    assert np.abs(x[7:7 + model.n_joints]).max() > 0.05  # the gait actually moved the spine


def test_mass_matrix_and_bias_vs_reference(model):
    from paper_2206_01683_b200 import dynamics as D
    r = model.robot()
    O = B.DynOracle(r)
    rng = np.random.default_rng(3)
    for _ in range(20):
        x = model.zero_state()
        x[:3] = rng.normal(size=3) * 0.1
        q = rng.normal(size=4)
        x[3:7] = q / np.linalg.norm(q)
        x[7:] = rng.normal(size=len(x) - 7) * 0.3
        st = model.unpack(x)
        assert _rel(O.mass_matrix(st), model.mass_matrix(x)) <= 1e-13
        g = (0.0, 0.0, -9.81)
        assert _rel(O.bias_forces(st, g), model.bias_forces(x, g)) <= 1e-13
        assert isinstance(st, D.JointState)


def test_skinning_restatement_vs_reference(model):
    import ref_models as RM
    S = RM.RefSamples(model, 0.02)
    P, N, A, W = model.samples(0.02)
    sk = model.skeleton()
    rng = np.random.default_rng(5)
    for trial in range(5):
        x = model.zero_state()
        x[:3] = rng.normal(size=3) * 0.2
        q = rng.normal(size=4)
        x[3:7] = q / np.linalg.norm(q)
        x[7:] = rng.normal(size=len(x) - 7) * 0.4
        pose = model.pose(x)
        pts, vel, nrm = B.skin_update(sk, pose, P, N, W)
        rp, rv, rn = S.update(x)
        assert _rel(pts, rp) <= 1e-13 and _rel(vel, rv) <= 1e-13 and _rel(nrm, rn) <= 1e-13
        f = rng.normal(size=(S.m, 3))
        valid = (rng.random(S.m) > 0.1).astype(np.int32)
        tau, st7 = B.skin_tau(sk, pose, P, W, f, valid, vel)
        rtau, rst = S.skinned_tau(x, f, valid)
        assert _rel(tau, rtau) <= 1e-13, trial
        assert _rel(st7, rst[:7]) <= 1e-13, trial


def test_empirical_backend_restatement_vs_reference(model):
    import ref_models as RM
    from paper_2206_01683_b200 import dynamics as D
    E = RM.EmpiricalRef(dt=0.004, substeps=4, rho=1000.0, spacing=0.02, k=40.0)
    E.add_robot(model, pos=(0.0, 0.0, 0.0), yaw=0.3)
    P, N, A, W = model.samples(0.02)
    r = model.robot()
    O = B.DynOracle(r)
    sk = model.skeleton()
    x0, _, _, bv = E.robot(0)
    st = model.unpack(x0)
    O.bladder_volume = bv
    worst = 0.0
    for k in range(100):
        act = _gait(r, k * 0.004)
        E.set_actuation(0, act)
        pose = model.pose(np.concatenate([st.base_pos, st.base_quat, st.q, st.v]))
        tau, stats = B.empirical_step(sk, pose, P, N, W, A, 40.0)
        O.robot_step(st, act, tau, 1000.0, (0.0, 0.0, -9.81), 0.004, 4)
        stable, _ = E.step()
        assert stable
        x, rtau, rst, _ = E.robot(0)
        worst = max(worst, _rel(np.concatenate([st.base_pos, st.base_quat, st.q, st.v]), x))
        if np.linalg.norm(rtau) > 0:
            assert _rel(tau, rtau) <= 1e-12, k
        assert np.allclose(stats[3:7], rst[3:7], rtol=1e-12, atol=1e-15), k
    assert worst <= 1e-12, worst
    assert isinstance(st, D.JointState)


@pytest.mark.parametrize("mutate,msg", [
    (lambda L: L.__setitem__((1, 0), 3.0), "parent must precede it"),
    (lambda L: L.__setitem__((2, 17), 0.0), "mass must be positive"),
    (lambda L: L.__setitem__((1, slice(14, 17)), 0.0), "zero joint axis"),
    (lambda L: L.__setitem__((3, 21), -1.0), "not positive definite"),
    (lambda L: L.__setitem__((3, 22), 0.5), "not symmetric"),
])
def test_validate_messages_match_reference(mutate, msg):
    """Skeleton::validate through the reference and through the product's
    fsg_dyn_create reject the same skeletons with the same message."""
    import ref_models as RM
    from paper_2206_01683_b200 import _abi
    m = RM.RefModel("koi")
    links = m.links.copy()
    mutate(links)
    L = B.ref()
    assert L.ref_skeleton_validate(len(links), B.dptr(np.ascontiguousarray(links))) == 1
    ref_msg = L.ref_robot_last_error().decode()
    assert msg in ref_msg
    bad = RM.RefModel("koi")
    bad.links = links
    from paper_2206_01683_b200.dynamics import RobotBatch
    with pytest.raises(_abi.InputError) as e:
        RobotBatch(bad.robot(), 1)  # validation precedes any device work
    assert ref_msg.split(":")[-1].strip() in str(e.value)
