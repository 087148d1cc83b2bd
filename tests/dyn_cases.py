"""Robots of the reference's robot tests (test_robot.cpp:17-66), built with the
product's host types (paper_2206_01683_b200.dynamics) -- test infrastructure."""
from __future__ import annotations

import numpy as np

from paper_2206_01683_b200.dynamics import FIXED, FREE, REVOLUTE, Link, Robot

G = np.array([0.0, 0.0, -9.81])  # kGravity (test_robot.cpp:15)


def base_link(jt) -> Link:
    """test_robot.cpp:17-25"""
    return Link(parent=-1, joint=jt, mass=1.0, inertia_com=1e-3 * np.eye(3))


def make_chain(n_joints, link_len, link_mass, base, along_x, stiffness=0.0, damping=0.0) -> Robot:
    """Planar chain under the base, every joint about y (test_robot.cpp:29-56)."""
    links = [base_link(base)]
    step = np.array([link_len, 0, 0]) if along_x else np.array([0, 0, -link_len])
    for j in range(n_joints):
        i_rod = link_mass * link_len * link_len / 12.0
        inertia = np.diag([1e-7, i_rod, i_rod]) if along_x else np.diag([i_rod, i_rod, 1e-7])
        links.append(Link(parent=j, joint=REVOLUTE, joint_origin=np.zeros(3) if j == 0 else step.astype(float),
                          axis=np.array([0.0, 1.0, 0.0]), mass=link_mass, com=0.5 * step,
                          inertia_com=inertia, stiffness=stiffness, damping=damping, limit_lo=-3.0,
                          limit_hi=3.0, torque_limit=100.0))
    return Robot(links)


def free_body(inertia, mass=2.0) -> Robot:
    """test_robot.cpp:58-64"""
    l = base_link(FREE)
    l.mass = mass
    l.inertia_com = np.asarray(inertia, dtype=float)
    return Robot([l])


def fin_tree() -> Robot:
    """The branched tree of test_robot.cpp:157-169: 3-link chain plus two fins."""
    t = make_chain(3, 0.12, 0.1, FREE, True)
    for side in (0, 1):
        t.links.append(Link(parent=1, joint=REVOLUTE,
                            joint_origin=np.array([0.03, -0.04 if side else 0.04, 0.0]),
                            axis=np.array([1.0, 0.0, 0.0]), mass=0.02,
                            com=np.array([0.0, -0.03 if side else 0.03, 0.0]),
                            inertia_com=1e-6 * np.eye(3)))
    return t


def skewed_chain() -> Robot:
    """A floating chain with mounted joint rotations, unnormalised axes, a fixed
    link, stiff springs and hydrostatics: exercises every term of the step."""
    r = make_chain(4, 0.1, 0.08, FREE, True, 2.0, 0.05)
    c, s = np.cos(0.3), np.sin(0.3)
    r.links[2].joint_rotation = np.array([[c, -s, 0], [s, c, 0], [0, 0, 1.0]])
    r.links[3].axis = np.array([0.2, 1.5, 0.4])
    r.links[4].joint = FIXED
    r.links[1].limit_lo, r.links[1].limit_hi = -0.2, 0.25
    for l in r.links:
        l.displaced_volume = l.mass / 1050.0
        l.volume_centroid = np.asarray(l.com, dtype=float) + np.array([0.0, 0.0, 0.004])
    r.bladder.volume = 2e-6
    r.bladder.centroid = np.array([0.01, 0.0, 0.002])
    return r
