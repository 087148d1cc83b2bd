"""CPU: the empirical-drag restatement (oracle orc_empirical_step,
EmpiricalBackend::step surface work, empirical.hpp:74-100) checked against
the reference's own empirical tests, restated:

* test_empirical.cpp:34-51  tangential motion is free; a plate moving along
  its normal feels exactly -k A v n; a retreating face feels no suction;
* test_empirical.cpp:85-99  the drag is dissipative for rigid motion (100
  random velocities, power <= 0);
* and the virtual-work identity of the generalized force it produces
  (test_ib.cpp:215-249 applied to the drag forces).
"""
import math

import numpy as np
import pytest

from oracle import bind as B
from paper_2206_01683_b200.scenes import (forward_kinematics, koi_articulation, koi_body,
                                          pack_pose)

K = 35.0


class _Sk:
    def __init__(self, parent, dof, axis, floating, ndof):
        self.parent, self.dof_index, self.axis = parent, dof, np.asarray(axis)
        self.floating_base, self.n_dofs = floating, ndof


RIGID = _Sk([-1], [0], np.zeros((1, 3)), True, 6)


def _rigid_pose(v, omega=(0.0, 0.0, 0.0)):
    """One floating link at the identity, moving with (v, omega) in the world."""
    R = np.eye(3)[None]
    return pack_pose(R, np.zeros((1, 3)), np.array([omega]), np.array([v]), R, np.zeros((1, 3)))


def _plate(n, v, area):
    n = np.asarray(n, dtype=np.float64)
    tau, st = B.empirical_step(RIGID, _rigid_pose(v), np.zeros((1, 3)), n[None], np.ones((1, 1)),
                               np.array([area]), K)
    return tau, st


def test_tangential_motion_is_free():
    n = np.array([0.3, -0.8, 0.52])
    n = n / np.linalg.norm(n)
    tau, st = _plate(n, np.cross(n, [0.0, 1.0, 0.0]), 0.01)
    assert (st == 0).all() and (tau == 0).all()


def test_normal_drag_exact_and_no_suction():
    n = np.array([0.3, -0.8, 0.52])
    n = n / np.linalg.norm(n)
    area, speed = 0.02, 0.4
    _, st = _plate(n, speed * n, area)
    assert np.linalg.norm(st[3:6] + K * area * speed * n) < 1e-14
    assert (st[:3] == 0).all()
    _, st2 = _plate(-n, speed * n, area)
    assert (st2 == 0).all()


@pytest.fixture(scope="module")
def fish():
    body = koi_body(0.03)
    art = koi_articulation(body)
    R, p, _, _ = forward_kinematics(art, np.eye(3), np.zeros(3), np.zeros(art.n_dofs),
                                    np.zeros(art.n_links - 1))
    sk = _Sk(art.parent, art.dof_index, art.axis, True, art.n_dofs)
    return body, art, sk, (R, p)


def test_dissipative_for_rigid_motion(fish):
    body, art, sk, rest = fish
    r = np.random.default_rng(7)
    for _ in range(100):
        v = np.zeros(art.n_dofs)
        v[3:6] = r.normal(size=3)
        R, p, om, vo = forward_kinematics(art, np.eye(3), np.zeros(3), v, np.zeros(art.n_links - 1))
        _, st = B.empirical_step(sk, pack_pose(R, p, om, vo, *rest), body.rest, body.normals,
                                 art.weights, body.areas, 20.0)
        assert st[6] <= 0.0


def test_virtual_work_identity(fish):
    body, art, sk, rest = fish
    r = B.Rng(31)
    q = np.array([r.uniform(-0.4, 0.4) for _ in range(art.n_links - 1)])
    v = np.array([r.uniform(-0.8, 0.8) for _ in range(art.n_dofs)])
    R, p, om, vo = forward_kinematics(art, np.eye(3), np.array([0.1, 0.0, 0.0]), v, q)
    tau, st = B.empirical_step(sk, pack_pose(R, p, om, vo, *rest), body.rest, body.normals,
                               art.weights, body.areas, K)
    assert st[6] < 0.0
    assert abs(tau @ v - st[6]) < 1e-10 * abs(st[6])
