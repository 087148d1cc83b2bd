"""Device robot dynamics (fsg_dyn_*, csrc/fsg_dyn.cu) against the fp64
restatement (oracle/fsg_dyn_oracle.c, pinned by test_dyn_oracle.py).

Tolerance: the device and the oracle run the same fp64 operations in the same
order (no FMA contraction on either side) except sin/cos (CUDA's vs libm's,
<= 2 ulp apart), so one step agrees to rel <= 1e-12 and a damped trajectory of
hundreds of steps to rel <= 1e-9."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import bind as B
from paper_2206_01683_b200 import dynamics as D
from paper_2206_01683_b200._abi import DYN_MAX_DOFS, DYN_MAX_LINKS
from paper_2206_01683_b200.scenes import koi_articulation, koi_body
from dyn_cases import G, fin_tree, make_chain, skewed_chain

pytestmark = pytest.mark.gpu


def _koi():
    body = koi_body(0.01)
    return D.koi_robot(body, koi_articulation(body))


def _robots():
    return {"koi": _koi(), "skewed": skewed_chain(), "fins": fin_tree(),
            "pendulum": make_chain(2, 0.4, 0.25, D.FIXED, False, 0.5, 0.01)}


def _random_states(robot, E, seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(E):
        st = D.JointState.zero(robot)
        st.base_pos = rng.uniform(-0.2, 0.2, 3)
        st.base_quat = B.quat_exp(rng.uniform(-1.5, 1.5, 3)) if robot.floating_base else st.base_quat
        st.q = rng.uniform(-0.6, 0.6, robot.n_joints)
        st.v = rng.uniform(-1.0, 1.0, robot.n_dofs)
        out.append(st)
    return out


def _copy(st):
    return D.JointState(st.base_pos.copy(), st.base_quat.copy(), st.q.copy(), st.v.copy(), st.qdd.copy())


def _state_vec(st):
    return np.concatenate([st.base_pos, st.base_quat, st.q, st.v, st.qdd])


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name", ["koi", "skewed", "fins", "pendulum"])
def test_mass_matrix_and_bias_match_oracle(name):
    robot = _robots()[name]
    E = 37
    rb = D.RobotBatch(robot, E)
    sts = _random_states(robot, E, 1)
    rb.set_states(sts)
    M, c = rb.mass_matrix(G)
    O = B.DynOracle(robot)
    for e in range(E):
        assert _rel(M[e], O.mass_matrix(sts[e])) <= 1e-12
        assert _rel(c[e], O.bias_forces(sts[e], G)) <= 1e-12
        # test_robot.cpp:180's symmetry bound (the CRBA sums are not exactly symmetric)
        assert np.linalg.norm(M[e] - M[e].T) < 1e-10 * (1.0 + np.linalg.norm(M[e]))


@pytest.mark.parametrize("name", ["koi", "skewed", "fins", "pendulum"])
def test_one_robot_step_matches_oracle(name):
    robot = _robots()[name]
    E = 40
    rng = np.random.default_rng(2)
    rb = D.RobotBatch(robot, E)
    sts = _random_states(robot, E, 3)
    rb.set_states(sts)
    act = rng.uniform(-0.5, 0.5, (E, robot.n_joints))
    act[0, :] = 1e3  # clamped against torque_limit
    tau = rng.uniform(-0.05, 0.05, (E, robot.n_dofs))
    flags = rb.step(act, tau, 1000.0, G, 0.004, 4, None)
    got = rb.states()
    O = B.DynOracle(robot)
    for e in range(E):
        x = _copy(sts[e])
        fl = O.robot_step(x, act[e], tau[e], 1000.0, G, 0.004, 4, None)
        assert flags[e] == fl
        assert _rel(_state_vec(got[e]), _state_vec(x)) <= 1e-12
    if robot.n_joints:
        assert flags[0] & D.FSG_DYN_CLAMPED


def test_koi_trajectory_matches_oracle():
    """300 steps of a gait-driven, buoyancy-trimmed koi with integrate's own
    gravity (tests both gravity paths) and 4 substeps."""
    robot = _koi()
    E = 8
    rb = D.RobotBatch(robot, E)
    sts = _random_states(robot, E, 4)
    for st in sts:
        st.v *= 0.2
    rb.set_states(sts)
    O = B.DynOracle(robot)
    ref = [_copy(s) for s in sts]
    nj = robot.n_joints
    for k in range(300):
        t = k * 0.004
        act = np.array([[0.25 * np.sin(2 * np.pi * 2.0 * t - 0.8 * j + e) for j in range(nj)]
                        for e in range(E)])
        flags = rb.step(act, None, 1000.0, G, 0.004, 4, 0.1 * G)
        for e in range(E):
            assert O.robot_step(ref[e], act[e], None, 1000.0, G, 0.004, 4, 0.1 * G) == flags[e]
    got = rb.states()
    for e in range(E):
        assert _rel(_state_vec(got[e]), _state_vec(ref[e])) <= 1e-9


def test_envs_are_independent():
    """A batch of 64 equals each env stepped alone (bit-identical)."""
    robot = skewed_chain()
    E = 64
    rng = np.random.default_rng(7)
    sts = _random_states(robot, E, 8)
    act = rng.uniform(-0.3, 0.3, (E, robot.n_joints))
    rb = D.RobotBatch(robot, E)
    rb.set_states(sts)
    rb.step(act, None, 1000.0, G, 0.004, 2)
    all_ = rb.states()
    for e in (0, 17, 63):
        one = D.RobotBatch(robot, 1)
        one.set_states([sts[e]])
        one.step(act[e:e + 1], None, 1000.0, G, 0.004, 2)
        assert np.array_equal(_state_vec(one.states()[0]), _state_vec(all_[e]))


def test_step_device_equals_host_call():
    torch = pytest.importorskip("torch")
    robot = _koi()
    E = 16
    rng = np.random.default_rng(9)
    sts = _random_states(robot, E, 10)
    act = rng.uniform(-0.3, 0.3, (E, robot.n_joints))
    tau = rng.uniform(-0.02, 0.02, (E, robot.n_dofs))
    a, b = D.RobotBatch(robot, E), D.RobotBatch(robot, E)
    a.set_states(sts)
    b.set_states(sts)
    fa = a.step(act, tau, 1000.0, G, 0.004, 4)
    ta = torch.tensor(act, dtype=torch.float64, device="cuda")
    tt = torch.tensor(tau, dtype=torch.float64, device="cuda")
    fl = torch.zeros(E, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    b.step_device(ta, tt, 1000.0, G, 0.004, 4, flags=fl)
    sb = b.states()  # synchronises the handle's stream
    for x, y in zip(a.states(), sb):
        assert np.array_equal(_state_vec(x), _state_vec(y))
    assert np.array_equal(fl.cpu().numpy(), fa)


def test_nonfinite_state_is_flagged_not_raised():
    robot = skewed_chain()
    rb = D.RobotBatch(robot, 2)
    sts = _random_states(robot, 2, 11)
    sts[1].v[0] = np.nan
    rb.set_states(sts)
    flags = rb.step(np.zeros((2, robot.n_joints)), None, 1000.0, G, 0.004, 1)
    assert not flags[0] & D.FSG_DYN_NONFINITE
    assert flags[1] & D.FSG_DYN_NONFINITE


def test_poses_match_oracle_and_feed_skinning():
    robot = _koi()
    E = 5
    rb = D.RobotBatch(robot, E)
    sts = _random_states(robot, E, 12)
    rb.set_states(sts)
    rR, rp = D.rest_pose(robot)
    P = rb.poses(rR, rp)
    O = B.DynOracle(robot)
    for e in range(E):
        ref = O.pose(sts[e], rR, rp)
        assert _rel(P[e], ref) <= 1e-12


def test_bladder_change_matches_host_mirror():
    robot = _koi()
    rb = D.RobotBatch(robot, 3)
    b = [D.Bladder(**{k: getattr(robot.bladder, k) for k in
                      ("volume", "volume_min", "volume_max", "rate_bound")}) for _ in range(3)]
    for dv in ([5e-7, -2e-6, 1e-5], [1e-5, 1e-5, -1e-5]):
        vol = rb.change_bladder(np.array(dv))
        for e in range(3):
            b[e].apply_change(dv[e])
            assert vol[e] == b[e].volume


@pytest.mark.parametrize("E", [24, 300])
@pytest.mark.parametrize("name", ["koi", "fins"])
def test_warp_and_thread_kernels_are_bit_identical(name, E, monkeypatch):
    """The warp-per-env kernel (small batches) and the thread-per-env kernel
    (large batches) run the same arithmetic: identical states and flags.
    E = 24: the warp kernel's two-warp form (RNEA on a helper warp, batches
    up to 256 envs); E = 300: its one-warp form."""
    robot = _robots()[name]
    rng = np.random.default_rng(13)
    sts = _random_states(robot, E, 14)
    act = rng.uniform(-0.5, 0.5, (E, robot.n_joints))
    act[3, :] = 50.0
    tau = rng.uniform(-0.05, 0.05, (E, robot.n_dofs))
    out = []
    for wmax in ("4096", "0"):
        monkeypatch.setenv("FSG_DYN_WARP_MAX", wmax)
        rb = D.RobotBatch(robot, E)
        rb.set_states(sts)
        fl = [rb.step(act, tau, 1000.0, G, 0.004, 4, 0.3 * G) for _ in range(20)]
        out.append((np.stack([_state_vec(s) for s in rb.states()]), np.stack(fl)))
    # (the light fins blow up under this drive: NaNs must match too)
    assert np.array_equal(out[0][0], out[1][0], equal_nan=True)
    assert np.array_equal(out[0][1], out[1][1])


def test_batch_step_dynamic_equals_host_loop():
    """fsg_batch_step_dynamic (poses from the robot states on the device, the
    coupled step, tau_ext into the robot step, one call) equals the host-driven
    loop: RobotBatch.poses -> EnvBatch.step_skinned -> RobotBatch.step with the
    returned tau_ext -- bit for bit (fluid, statuses, robot states)."""
    from paper_2206_01683_b200 import EnvBatch, SessionConfig
    from skin_cases import init_fluid, skin_scene
    sc = skin_scene()
    E = 3
    robot = D.koi_robot(sc.bodies[0], sc.articulations()[0])
    rR, rp = D.rest_pose(robot)
    cfg = SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                        frame_mode=sc.frame_mode, precision="fp32", max_markers=sc.m)
    rho, u = init_fluid(sc)
    A, Bt = EnvBatch(cfg, E), EnvBatch(cfg, E)
    RA, RB = D.RobotBatch(robot, E), D.RobotBatch(robot, E)
    sts = _random_states(robot, E, 21)
    for st in sts:
        st.base_pos[:] = 0.0
        st.v *= 0.1
        st.q *= 0.3
    for bt in (A, Bt):
        for s in bt.envs:
            s.initialize(rho, u)
            s.set_skin(*sc.skin())
    RA.set_states(sts)
    RB.set_states(sts)
    RB.set_rest(rR, rp)
    rng = np.random.default_rng(22)
    for k in range(6):
        frames = np.stack([sc.frame(k + 3 * e).packed() for e in range(E)])
        act = rng.uniform(-0.2, 0.2, (E, robot.n_joints))
        sa, taus, _ = A.step_skinned(frames, RA.poses(rR, rp))
        fa = RA.step(act, np.stack(taus), sc.rho, G, sc.dt, 4)
        sb, fb, packed = Bt.step_dynamic(RB, act, frames, sc.rho, G, sc.dt, 4)
        stb = D.unpack_states(packed, robot.n_joints, robot.n_dofs)
        assert np.array_equal(fa, fb)
        for e in range(E):
            assert sa[e].min_f == sb[e].min_f and sa[e].stable() == sb[e].stable()
        for x, y in zip(RA.states(), stb):
            assert np.array_equal(_state_vec(x), _state_vec(y))
        assert np.abs(np.stack(taus)).max() > 0.0
    for e in range(E):
        assert np.array_equal(A.envs[e].get_f(), Bt.envs[e].get_f())
    A.close()
    Bt.close()


def test_batch_step_dynamic_rejects_mismatches():
    from paper_2206_01683_b200 import EnvBatch, FsgError, InputError, SessionConfig
    from skin_cases import skin_scene
    sc = skin_scene()
    robot = D.koi_robot(sc.bodies[0], sc.articulations()[0])
    cfg = SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                        frame_mode=sc.frame_mode, precision="fp32", max_markers=sc.m)
    b = EnvBatch(cfg, 2)
    act = np.zeros((2, robot.n_joints))
    with pytest.raises(InputError, match="robots for"):
        b.step_dynamic(D.RobotBatch(robot, 3), np.zeros((3, robot.n_joints)))
    with pytest.raises(FsgError, match="fsg_dyn_set_rest"):
        b.step_dynamic(D.RobotBatch(robot, 2), act)
    rb = D.RobotBatch(robot, 2)
    rb.set_rest(*D.rest_pose(robot))
    with pytest.raises(FsgError, match="no single skinned body"):
        b.step_dynamic(rb, act)
    for s in b.envs:
        s.set_skin(*sc.skin())
    st, fl, packed = b.step_dynamic(rb, act)  # now well-formed
    assert all(x.stable() for x in st) and packed.shape == (2, 7 + DYN_MAX_LINKS + 2 * DYN_MAX_DOFS)
    b.close()


@pytest.mark.parametrize("E,wmax", [(4, "4096"), (300, "4096"), (4, "0")])
def test_not_spd_env_stops_alone(E, wmax, monkeypatch):
    """A NaN joint angle makes that env's mass matrix NaN: the Cholesky stops
    it with FSG_DYN_NOT_SPD (the reference's NumericalError) at the first
    substep -- in the warp kernel's two-warp form (the helper warp must leave
    its barrier loop), its one-warp form and the thread kernel -- while the
    other envs step on, identical to a batch without the bad env."""
    monkeypatch.setenv("FSG_DYN_WARP_MAX", wmax)
    robot = _koi()
    sts = _random_states(robot, E, 21)
    act = np.zeros((E, robot.n_joints))
    tau = np.zeros((E, robot.n_dofs))
    good = D.RobotBatch(robot, E)
    good.set_states(sts)
    fl_good = good.step(act, tau, 1000.0, G, 0.004, 4)
    bad_sts = list(sts)
    bad = D.JointState.zero(robot)
    bad.q[0] = np.nan
    bad_sts[1] = bad
    rb = D.RobotBatch(robot, E)
    rb.set_states(bad_sts)
    fl = rb.step(act, tau, 1000.0, G, 0.004, 4)
    assert fl[1] & D.FSG_DYN_NOT_SPD
    keep = [e for e in range(E) if e != 1]
    assert np.array_equal(fl[keep], fl_good[keep])
    a = np.stack([_state_vec(s) for s in rb.states()])[keep]
    b = np.stack([_state_vec(s) for s in good.states()])[keep]
    assert np.array_equal(a, b)
    rb.close()
    good.close()
