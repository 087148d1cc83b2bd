"""CPU: the skinning restatement (oracle/fsg_oracle.c orc_update_samples /
orc_skin_tau) checked against the reference's OWN tests for these functions,
restated with their tolerances:

* test_sampling.cpp:45-110  "skinning identities" (identity pose, rigid
  translation, fully owned vertices rotate with their joint, rigid-motion
  equivariance);
* test_sampling.cpp:112-138 "skin velocities match finite-differenced positions";
* test_sampling.cpp:178-193 "sample velocities agree with rigid-body motion";
* test_ib.cpp:215-249      "virtual work identity: sample forces vs generalized forces".

These pin the restatement that the GPU parity tests (test_skin_gpu.py)
compare against bit for bit.  The reference headers themselves need
dynamic-size Eigen and do not compile against the oracle's stand-in
(SURVEY.md §8(c)).
"""
import math

import numpy as np
import pytest

from oracle import bind as B
from paper_2206_01683_b200.scenes import (forward_kinematics, koi_articulation, koi_body,
                                          pack_pose, _rotz)


def _quat_R(v):
    """quat_exp(v) rotation (types.hpp)."""
    th = np.linalg.norm(v)
    a = v / th if th > 0 else np.array([0.0, 0.0, 1.0])
    c, s = math.cos(th), math.sin(th)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + s * K + (1 - c) * K @ K


@pytest.fixture(scope="module")
def fish():
    body = koi_body(0.02)
    art = koi_articulation(body)
    R, p, _, _ = forward_kinematics(art, np.eye(3), np.zeros(3), np.zeros(art.n_dofs),
                                    np.zeros(art.n_links - 1))
    return body, art, (R, p)


class _Sk:
    def __init__(self, art):
        self.parent, self.dof_index, self.axis = art.parent, art.dof_index, art.axis
        self.floating_base, self.n_dofs = art.floating_base, art.n_dofs


def _skin(fish, base_R, base_p, v, q):
    body, art, rest = fish
    R, p, om, vo = forward_kinematics(art, base_R, base_p, v, q)
    P = pack_pose(R, p, om, vo, *rest)
    return B.skin_update(_Sk(art), P, body.rest, body.normals, art.weights), P, (R, p, om, vo)


def test_weights_partition(fish):
    _, art, _ = fish
    assert np.allclose(art.weights.sum(1), 1.0, atol=1e-12)
    assert (art.weights >= 0).all() and ((art.weights > 0).sum(1) <= 4).all()


def test_identity_pose_returns_rest(fish):
    body, art, _ = fish
    (pts, vel, nrm), _, _ = _skin(fish, np.eye(3), np.zeros(3), np.zeros(art.n_dofs),
                                  np.zeros(art.n_links - 1))
    assert np.linalg.norm(pts - body.rest, axis=1).max() < 1e-14
    assert (np.linalg.norm(vel, axis=1) == 0.0).all()


def test_rigid_translation(fish):
    body, art, _ = fish
    shift = np.array([0.3, -0.2, 0.15])
    (pts, _, _), _, _ = _skin(fish, np.eye(3), shift, np.zeros(art.n_dofs), np.zeros(art.n_links - 1))
    assert np.linalg.norm(pts - body.rest - shift, axis=1).max() < 1e-14


def test_owned_vertices_rotate_with_joint(fish):
    body, art, _ = fish
    q = np.zeros(art.n_links - 1)
    q[-1] = math.pi / 6
    (pts, _, _), _, (R, p, _, _) = _skin(fish, np.eye(3), np.zeros(3), np.zeros(art.n_dofs), q)
    last = art.n_links - 1
    rz = _rotz(math.pi / 6)
    own = art.weights[:, last] == 1.0
    assert own.sum() > 10
    exp = p[last] + (body.rest[own] - p[last]) @ rz.T
    assert np.linalg.norm(pts[own] - exp, axis=1).max() < 1e-13


def test_rigid_motion_equivariance(fish):
    body, art, _ = fish
    r = B.Rng(5)
    q = np.array([r.uniform(-0.5, 0.5) for _ in range(art.n_links - 1)])
    (pts, _, _), _, _ = _skin(fish, np.eye(3), np.zeros(3), np.zeros(art.n_dofs), q)
    rot = _quat_R(np.array([0.4, -0.3, 1.1]))
    shift = np.array([0.2, 0.7, -0.4])
    (pts2, _, _), _, _ = _skin(fish, rot, shift, np.zeros(art.n_dofs), q)
    assert np.linalg.norm(pts2 - (pts @ rot.T + shift), axis=1).max() < 1e-12


def test_rigid_body_velocity(fish):
    body, art, _ = fish
    v = np.zeros(art.n_dofs)
    v[:3] = (0.0, 0.0, 1.3)
    v[3:6] = (0.5, 0.0, 0.0)
    (pts, vel, _), _, _ = _skin(fish, np.eye(3), np.zeros(3), v, np.zeros(art.n_links - 1))
    exp = np.array([0.5, 0.0, 0.0]) + np.cross(np.array([0.0, 0.0, 1.3]), pts)
    assert np.linalg.norm(vel - exp, axis=1).max() < 1e-12


def test_velocity_matches_finite_difference(fish):
    body, art, _ = fish
    r = B.Rng(9)
    q = np.array([r.uniform(-0.3, 0.3) for _ in range(art.n_links - 1)])
    v = np.array([r.uniform(-1.0, 1.0) for _ in range(art.n_dofs)])
    R0 = _quat_R(np.array([0.1, -0.2, 0.3]))
    p0 = np.array([0.05, 0.0, -0.02])
    (pos0, vel0, _), _, _ = _skin(fish, R0, p0, v, q)
    dt = 1e-6
    R1 = R0 @ _quat_R(v[:3] * dt)
    p1 = p0 + R0 @ v[3:6] * dt
    (pos1, _, _), _, _ = _skin(fish, R1, p1, v, q + v[6:] * dt)
    fd = (pos1 - pos0) / dt
    assert (np.linalg.norm(fd - vel0, axis=1) < 5e-4 * np.maximum(1.0, np.linalg.norm(vel0, axis=1))).all()


def test_virtual_work_identity(fish):
    body, art, _ = fish
    r = B.Rng(31)
    q = np.array([r.uniform(-0.4, 0.4) for _ in range(art.n_links - 1)])
    v = np.array([r.uniform(-0.8, 0.8) for _ in range(art.n_dofs)])
    R0 = _quat_R(np.array([r.uniform(-1, 1) for _ in range(3)]))
    (pts, vel, _), P, _ = _skin(fish, R0, np.array([0.3, -0.1, 0.2]), v, q)
    f = np.random.default_rng(31).normal(size=(body.m, 3))
    # orc_skin_tau applies -f per marker (session.hpp:139-140): pass -f to get J^T f
    tau, stats = B.skin_tau(_Sk(art), P, body.rest, art.weights, -f, np.ones(body.m, np.int32), vel)
    p_samples = float((f * vel).sum())
    assert abs(p_samples - tau @ v) < 1e-8 * max(1.0, abs(p_samples))
    assert stats[6] == pytest.approx(p_samples, rel=1e-12)  # power_on_body = sum(-(-f)).v
    assert np.allclose(stats[:3], -f.sum(0)) and np.allclose(stats[3:6], f.sum(0))


def test_invalid_markers_contribute_nothing(fish):
    body, art, _ = fish
    (pts, vel, _), P, _ = _skin(fish, np.eye(3), np.zeros(3), np.zeros(art.n_dofs),
                                np.zeros(art.n_links - 1))
    f = np.ones((body.m, 3))
    tau, stats = B.skin_tau(_Sk(art), P, body.rest, art.weights, f, np.zeros(body.m, np.int32), vel)
    assert (tau == 0).all() and (stats == 0).all()
