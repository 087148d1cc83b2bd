"""Pins the fp64 dynamics restatement (oracle/fsg_dyn_oracle.c) with the
reference's own robot tests (test_robot.cpp:69-343), restated; quat_exp is
checked bit-for-bit against the reference's types.hpp compiled in oracle/_ref.
CPU only."""
from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import bind as B
from paper_2206_01683_b200.dynamics import FIXED, FREE, Bladder, JointState, Robot
from dyn_cases import G, fin_tree, free_body, make_chain


def test_quat_exp_matches_reference():
    if not B.have_ref():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(5)
    for w in list(rng.uniform(-2, 2, (200, 3))) + [np.array([1e-13, -2e-13, 0.0]), np.zeros(3)]:
        q, r = B.quat_exp(w), np.zeros(4)
        B.ref().ref_quat_exp(B.dptr(B.d3(w)), B.dptr(r))
        assert np.array_equal(q, r)


def test_free_single_link_at_rest_has_zero_acceleration():
    """test_robot.cpp:69-74"""
    s = free_body(np.eye(3) * 0.01)
    O = B.DynOracle(s)
    qdd = O.forward_dynamics(JointState.zero(s), np.zeros(6), np.zeros(6))
    assert np.linalg.norm(qdd) < 1e-12


def test_free_rigid_body_conserves_momentum_while_tumbling():
    """test_robot.cpp:76-111"""
    s = free_body(np.diag([0.02, 0.013, 0.008]), 1.7)
    O = B.DynOracle(s)
    st = JointState.zero(s)
    st.v = np.array([1.2, -0.7, 0.9, 0.3, 0.1, -0.2])
    inertia = s.links[0].inertia_com

    def momentum(x):
        r = B.quat_to_R(x.base_quat)
        return s.links[0].mass * (r @ x.v[3:6]), r @ (inertia @ x.v[:3])

    qdd = O.forward_dynamics(st, np.zeros(6), np.zeros(6))
    world_acc = B.quat_to_R(st.base_quat) @ (qdd[3:6] + np.cross(st.v[:3], st.v[3:6]))
    assert np.linalg.norm(world_acc) < 1e-12

    def drift(dt, steps):
        x = JointState(st.base_pos.copy(), st.base_quat.copy(), st.q.copy(), st.v.copy(), st.qdd.copy())
        lin0, ang0 = momentum(x)
        for _ in range(steps):
            O.integrate(x, [], np.zeros(6), dt, 1)
        lin1, ang1 = momentum(x)
        return np.linalg.norm(lin1 - lin0) / np.linalg.norm(lin0) + \
            np.linalg.norm(ang1 - ang0) / np.linalg.norm(ang0)

    coarse, fine = drift(1e-3, 2000), drift(1e-4, 20000)
    assert fine < 0.2 * coarse
    assert fine < 5e-4


def test_pendulum_oscillates_at_the_analytic_frequency():
    """test_robot.cpp:113-139"""
    ln, mass = 0.5, 0.3
    s = make_chain(1, ln, mass, FIXED, False)
    O = B.DynOracle(s)
    st = JointState.zero(s)
    st.q[0] = 0.05
    period = 2.0 * math.pi / math.sqrt(3.0 * 9.81 / (2.0 * ln))
    dt = 1e-4
    crossings, prev = [], st.q[0]
    for k in range(int(10.5 * period / dt)):
        O.integrate(st, np.zeros(1), np.zeros(1), dt, 1, G)
        if prev < 0.0 <= st.q[0]:
            crossings.append((k - prev / (st.q[0] - prev)) * dt)
        prev = st.q[0]
    assert len(crossings) >= 10
    measured = (crossings[-1] - crossings[0]) / (len(crossings) - 1)
    assert abs(measured / period - 1.0) < 0.005


def test_undamped_double_pendulum_conserves_energy():
    """test_robot.cpp:141-152 (10 s at dt = 1e-4)"""
    s = make_chain(2, 0.4, 0.25, FIXED, False)
    O = B.DynOracle(s)
    st = JointState.zero(s)
    st.q = np.array([0.8, 0.4])
    e0 = O.mechanical_energy(st, G)
    for _ in range(100000):
        O.integrate(st, np.zeros(2), np.zeros(2), 1e-4, 1, G)
    e1 = O.mechanical_energy(st, G)
    assert abs(e1 - e0) / max(abs(e0), 1e-6) < 0.01


def test_mass_matrix_spd_across_random_poses():
    """test_robot.cpp:154-185 (Rng(42), 500 poses each of the chain and the fin tree)"""
    chain = make_chain(7, 0.1, 0.08, FREE, True)
    rng = B.Rng(42)
    for s in (chain, fin_tree()):
        O = B.DynOracle(s)
        for _ in range(500):
            st = JointState.zero(s)
            for j in range(len(st.q)):
                st.q[j] = rng.uniform(-1.2, 1.2)
            st.base_quat = B.quat_exp([rng.uniform(-2, 2), rng.uniform(-2, 2), rng.uniform(-2, 2)])
            m = O.mass_matrix(st)
            assert np.linalg.norm(m - m.T) < 1e-10 * (1.0 + np.linalg.norm(m))
            x = np.zeros(s.n_dofs)
            assert B.oracle().orc_llt_solve(s.n_dofs, B.dptr(np.ascontiguousarray(m).reshape(-1)),
                                            B.dptr(np.ones(s.n_dofs)), B.dptr(x)) == 1


def test_internal_forces_rest_restoring_clamping():
    """test_robot.cpp:187-224"""
    s = make_chain(3, 0.2, 0.1, FIXED, True, 2.0, 0.05)
    O = B.DynOracle(s)
    st = JointState.zero(s)
    tau, _ = O.internal_forces(st, np.zeros(3))
    assert np.linalg.norm(tau) == 0.0
    st.q[1] = 0.3
    tau, _ = O.internal_forces(st, np.zeros(3))
    assert tau[1] < 0.0 and tau[0] == 0.0
    st.q[1] = -0.3
    assert O.internal_forces(st, np.zeros(3))[0][1] > 0.0
    st.q[1] = 0.0
    tau, clamped = O.internal_forces(st, np.array([1e4, 0.0, 0.0]))
    assert clamped and tau[0] == pytest.approx(s.links[1].torque_limit)
    sf = make_chain(2, 0.2, 0.1, FREE, True, 2.0, 0.05)
    stf = JointState.zero(sf)
    stf.q = np.array([0.4, -0.2])
    tau, _ = B.DynOracle(sf).internal_forces(stf, np.array([0.3, 0.1]))
    assert np.linalg.norm(tau[:6]) == 0.0


def test_driven_chain_matches_linearized_frequency_response():
    """test_robot.cpp:226-267 (30 s at dt = 1e-4)"""
    nj, ln, mass, k_spring, c_damp = 3, 0.15, 0.1, 2.0, 0.05
    s = make_chain(nj, ln, mass, FIXED, True, k_spring, c_damp)
    for i in range(1, nj + 1):
        s.links[i].com = np.array([ln, 0, 0])
        s.links[i].inertia_com = 1e-8 * np.eye(3)
    m0 = np.zeros((nj, nj))
    for j in range(nj):
        for l in range(nj):
            for k in range(max(j, l), nj):
                m0[j, l] += mass * (k + 1 - j) * (k + 1 - l) * ln * ln
    amp, w = 0.002, 3.0
    a = (-w * w * m0).astype(complex)
    a[np.diag_indices(nj)] += complex(k_spring, w * c_damp)
    qhat = np.linalg.solve(a, np.full(nj, amp, dtype=complex))
    O = B.DynOracle(s)
    st = JointState.zero(s)
    dt, t_total, t = 1e-4, 30.0, 0.0
    lo, hi = np.full(nj, 1e9), np.full(nj, -1e9)
    while t < t_total:
        O.integrate(st, np.full(nj, amp * math.sin(w * t)), np.zeros(nj), dt, 1)
        if t > 0.75 * t_total:
            lo, hi = np.minimum(lo, st.q), np.maximum(hi, st.q)
        t += dt
    measured = 0.5 * (hi - lo)
    assert np.all(np.abs(measured / np.abs(qhat) - 1.0) < 0.05)


def test_joint_limits_clamp_position():
    """test_robot.cpp:269-279"""
    s = make_chain(1, 0.2, 0.1, FIXED, True)
    s.links[1].limit_hi, s.links[1].limit_lo = 0.5, -0.5
    O = B.DynOracle(s)
    st = JointState.zero(s)
    for _ in range(20000):
        O.integrate(st, np.array([50.0]), np.zeros(1), 1e-4, 1)
    assert -0.5 - 1e-9 <= st.q[0] <= 0.5 + 1e-9


def test_buoyancy_balances_gravity_at_neutral_trim():
    """test_robot.cpp:281-330"""
    rho = 1000.0
    s = make_chain(2, 0.2, 0.5, FREE, True)
    for l in s.links:
        l.displaced_volume = l.mass / rho
        l.volume_centroid = np.asarray(l.com, dtype=float).copy()
    st = JointState.zero(s)
    st.q = np.array([0.3, -0.5])
    st.base_quat = B.quat_exp([0.2, 0.1, 0.4])
    assert np.linalg.norm(B.DynOracle(s).buoyancy_gravity_forces(st, rho, G, 0.0)) < 1e-10
    for l in s.links:
        l.displaced_volume = l.mass / 1080.0
    assert s.neutral_trim_volume(rho) > 0.0
    mono = Robot([s.links[0]])
    mono.links[0].mass = 1.08
    mono.links[0].displaced_volume = 1.08 / 1080.0
    mono.links[0].volume_centroid = np.asarray(mono.links[0].com, dtype=float).copy()
    b2 = Bladder(volume=mono.neutral_trim_volume(rho), volume_max=1.0)
    mono.bladder = b2
    st2 = JointState.zero(mono)
    O = B.DynOracle(mono)
    assert np.linalg.norm(O.buoyancy_gravity_forces(st2, rho, G, b2.volume)) < 1e-10
    dv = 0.1 * b2.volume
    tau2 = O.buoyancy_gravity_forces(st2, rho, G, b2.volume + dv)
    assert abs(tau2[5] - rho * 9.81 * dv) < 1e-10


def test_bladder_volume_and_rate_stay_bounded():
    """test_robot.cpp:332-344 (the host mirror's Bladder.apply_change)"""
    b = Bladder(volume=1e-5, volume_min=0.0, volume_max=2e-5, rate_bound=1e-6)
    b.apply_change(5e-6)
    assert b.volume == pytest.approx(1.1e-5)
    for _ in range(100):
        b.apply_change(1e-6)
    assert b.volume == pytest.approx(2e-5)
    for _ in range(100):
        b.apply_change(-1e-6)
    assert b.volume == pytest.approx(0.0, abs=1e-18)


# ---- the boundary's CPU-side behaviour (no device needed) --------------------
def _cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.parametrize("mutate,msg", [
    (lambda r: setattr(r.links[0], "joint", 1), "root joint must be free or fixed"),
    (lambda r: setattr(r.links[2], "parent", 2), "parent must precede it"),
    (lambda r: setattr(r.links[1], "joint", 0), "only the root may be free"),
    (lambda r: setattr(r.links[1], "axis", np.zeros(3)), "zero joint axis"),
    (lambda r: setattr(r.links[1], "limit_lo", 4.0), "joint limits inverted"),
    (lambda r: setattr(r.links[2], "mass", 0.0), "mass must be positive"),
    (lambda r: setattr(r.links[1], "inertia_com", np.array([[1, 0.1, 0], [0, 1, 0], [0, 0, 1.0]])),
     "not symmetric"),
    (lambda r: setattr(r.links[1], "inertia_com", np.diag([1.0, -1.0, 1.0])), "not positive definite"),
])
def test_skeleton_validate_messages(mutate, msg):
    """Skeleton::validate (skeleton.hpp:95-118; test_robot.cpp:346-363) through fsg_dyn_create."""
    from paper_2206_01683_b200 import _abi
    from paper_2206_01683_b200.dynamics import RobotBatch
    r = make_chain(3, 0.1, 0.1, FREE, True)
    mutate(r)
    with pytest.raises(_abi.InputError, match=msg):
        RobotBatch(r, 4)


@pytest.mark.skipif(_cuda_available(), reason="checks the no-GPU failure path")
def test_dyn_no_cpu_fallback_without_gpu():
    from paper_2206_01683_b200 import _abi
    from paper_2206_01683_b200.dynamics import RobotBatch
    with pytest.raises(_abi.FsgError, match="no CUDA device"):
        RobotBatch(make_chain(2, 0.1, 0.1, FREE, True), 4)
