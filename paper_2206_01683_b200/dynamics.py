"""Articulated robot dynamics for a batch of envs on the device.

Host mirror of the reference's robot types and of the robot half of
``CoupledSession::step`` (session.hpp:169-175), over the C ABI ``fsg_dyn_*``
(include/fsg.h; kernels in csrc/fsg_dyn.cu):

* ``Link`` / ``Bladder`` / ``Robot``  -- robot::Link, Bladder, Skeleton
  (skeleton.hpp:16-93), same field names and meaning;
* ``JointState``                      -- robot::JointState (skeleton.hpp:138-150);
* ``RobotBatch``                      -- E robots of one skeleton on one device:
  ``step`` = buoyancy_gravity_forces (dynamics.hpp:237-255) on the pre-step
  kinematics + integrate (dynamics.hpp:259-289) for every env in one launch;
  ``mass_matrix`` (CRBA + RNEA probes), ``poses`` (forward kinematics +
  BoneTransforms::of for the device skinning), ``change_bladder``
  (Bladder::apply_change).

Invalid skeletons raise ``InputError`` with Skeleton::validate's messages; a
mass matrix that is not positive definite (the reference's NumericalError,
dynamics.hpp:208-210) is reported per env as ``FSG_DYN_NOT_SPD``.  There is no
CPU fallback: without libfsg.so or a device every call fails loudly.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._abi import (DYN_MAX_DOFS, DYN_MAX_LINKS, FSG_DYN_CLAMPED, FSG_DYN_NONFINITE,  # noqa: F401
                   FSG_DYN_NOT_SPD, FSG_JOINT_FIXED, FSG_JOINT_FREE, FSG_JOINT_REVOLUTE,
                   fsg_body_pose, fsg_joint_state, fsg_robot)

FREE, REVOLUTE, FIXED = FSG_JOINT_FREE, FSG_JOINT_REVOLUTE, FSG_JOINT_FIXED


def _v(x, n=3):
    return np.asarray(x, dtype=np.float64).reshape(n)


@dataclass
class Link:
    """robot::Link (skeleton.hpp:16-36)."""

    parent: int = -1
    joint: int = REVOLUTE
    joint_origin: np.ndarray = field(default_factory=lambda: np.zeros(3))
    joint_rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    axis: np.ndarray = field(default_factory=lambda: np.array([0.0, 0.0, 1.0]))
    mass: float = 0.0
    com: np.ndarray = field(default_factory=lambda: np.zeros(3))
    inertia_com: np.ndarray = field(default_factory=lambda: np.eye(3))
    stiffness: float = 0.0
    damping: float = 0.0
    q_rest: float = 0.0
    limit_lo: float = -1.5
    limit_hi: float = 1.5
    torque_limit: float = 1.0
    displaced_volume: float = 0.0
    volume_centroid: np.ndarray = field(default_factory=lambda: np.zeros(3))


@dataclass
class Bladder:
    """robot::Bladder (skeleton.hpp:38-52)."""

    volume: float = 0.0
    volume_min: float = 0.0
    volume_max: float = 0.0
    rate_bound: float = 0.0
    centroid: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def apply_change(self, dv: float) -> None:
        self.volume = min(max(self.volume + min(max(dv, -self.rate_bound), self.rate_bound),
                              self.volume_min), self.volume_max)


@dataclass
class Robot:
    """robot::Skeleton + its Bladder (skeleton.hpp:54-93)."""

    links: list
    bladder: Bladder = field(default_factory=Bladder)

    @property
    def n_links(self) -> int:
        return len(self.links)

    @property
    def floating_base(self) -> bool:
        return bool(self.links) and self.links[0].joint == FREE

    @property
    def n_joints(self) -> int:
        return sum(1 for l in self.links[1:] if l.joint == REVOLUTE)

    @property
    def n_dofs(self) -> int:
        return (6 if self.floating_base else 0) + self.n_joints

    def dof_index(self, i: int) -> int:
        if i == 0:
            return 0 if self.floating_base else -1
        if self.links[i].joint != REVOLUTE:
            return -1
        return (6 if self.floating_base else 0) + sum(
            1 for k in range(1, i) if self.links[k].joint == REVOLUTE)

    def total_mass(self) -> float:
        return float(sum(l.mass for l in self.links))

    def total_displaced_volume(self) -> float:
        return float(sum(l.displaced_volume for l in self.links))

    def neutral_trim_volume(self, rho_fluid: float) -> float:
        return self.total_mass() / rho_fluid - self.total_displaced_volume()

    def to_struct(self) -> fsg_robot:
        if self.n_links > DYN_MAX_LINKS:
            raise _abi.InputError(_abi.FSG_EINPUT, f"skeleton has {self.n_links} links "
                                                   f"(max {DYN_MAX_LINKS})")
        r = fsg_robot()
        r.n_links = self.n_links
        for i, l in enumerate(self.links):
            s = r.links[i]
            s.parent, s.joint = int(l.parent), int(l.joint)
            s.joint_origin[:] = _v(l.joint_origin)
            s.joint_rotation[:] = _v(l.joint_rotation, 9)
            s.axis[:] = _v(l.axis)
            s.mass = float(l.mass)
            s.com[:] = _v(l.com)
            s.inertia_com[:] = _v(l.inertia_com, 9)
            s.stiffness, s.damping, s.q_rest = float(l.stiffness), float(l.damping), float(l.q_rest)
            s.limit_lo, s.limit_hi = float(l.limit_lo), float(l.limit_hi)
            s.torque_limit = float(l.torque_limit)
            s.displaced_volume = float(l.displaced_volume)
            s.volume_centroid[:] = _v(l.volume_centroid)
        b = self.bladder
        r.bladder_volume, r.bladder_volume_min = float(b.volume), float(b.volume_min)
        r.bladder_volume_max, r.bladder_rate_bound = float(b.volume_max), float(b.rate_bound)
        r.bladder_centroid[:] = _v(b.centroid)
        return r


@dataclass
class JointState:
    """robot::JointState (skeleton.hpp:138-150); base_quat is (w, x, y, z)."""

    base_pos: np.ndarray
    base_quat: np.ndarray
    q: np.ndarray
    v: np.ndarray
    qdd: np.ndarray

    @staticmethod
    def zero(robot: Robot) -> "JointState":
        return JointState(np.zeros(3), np.array([1.0, 0.0, 0.0, 0.0]), np.zeros(robot.n_joints),
                          np.zeros(robot.n_dofs), np.zeros(robot.n_dofs))

    def to_struct(self) -> fsg_joint_state:
        s = fsg_joint_state()
        s.base_pos[:] = _v(self.base_pos)
        s.base_quat[:] = _v(self.base_quat, 4)
        nj, nd = len(self.q), len(self.v)
        s.q[:nj] = np.asarray(self.q, dtype=np.float64)
        s.v[:nd] = np.asarray(self.v, dtype=np.float64)
        s.qdd[:nd] = np.asarray(self.qdd, dtype=np.float64)
        return s

    @staticmethod
    def from_struct(s: fsg_joint_state, nj: int, nd: int) -> "JointState":
        return JointState(np.array(s.base_pos[:]), np.array(s.base_quat[:]), np.array(s.q[:nj]),
                          np.array(s.v[:nd]), np.array(s.qdd[:nd]))


def unpack_states(packed, n_joints: int, n_dofs: int) -> list:
    """Packed fsg_joint_state rows ([E, 7 + DYN_MAX_LINKS + 2 DYN_MAX_DOFS], EnvBatch.step_dynamic)
    -> JointStates."""
    L, Dm = DYN_MAX_LINKS, DYN_MAX_DOFS
    out = []
    for r in np.asarray(packed, dtype=np.float64).reshape(-1, 7 + L + 2 * Dm):
        out.append(JointState(r[0:3].copy(), r[3:7].copy(), r[7:7 + n_joints].copy(),
                              r[7 + L:7 + L + n_dofs].copy(), r[7 + L + Dm:7 + L + Dm + n_dofs].copy()))
    return out


class RobotBatch:
    """E robots of one skeleton on one device (fsg_dyn_*)."""

    def __init__(self, robot: Robot, n_envs: int, device: int = 0):
        L = _abi.lib()
        self.robot = robot
        self.n_envs = int(n_envs)
        self._struct = robot.to_struct()
        h = C.c_void_p()
        _abi.check(L.fsg_dyn_create(C.byref(self._struct), self.n_envs, int(device), C.byref(h)),
                   dyn=True)
        self._h = h
        self.n_dofs = int(L.fsg_dyn_n_dofs(h))
        self.n_joints = int(L.fsg_dyn_n_joints(h))

    def close(self) -> None:
        if getattr(self, "_h", None):
            _abi.lib().fsg_dyn_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- state ---------------------------------------------------------------
    def set_states(self, states) -> None:
        arr = (fsg_joint_state * self.n_envs)(*[s.to_struct() for s in states])
        _abi.check(_abi.lib().fsg_dyn_set_state(self._h, arr), dyn=True)

    def states(self) -> list:
        arr = (fsg_joint_state * self.n_envs)()
        _abi.check(_abi.lib().fsg_dyn_get_state(self._h, arr), dyn=True)
        return [JointState.from_struct(arr[e], self.n_joints, self.n_dofs)
                for e in range(self.n_envs)]

    def change_bladder(self, dv) -> np.ndarray:
        dv = np.ascontiguousarray(np.broadcast_to(np.asarray(dv, dtype=np.float64), (self.n_envs,)))
        out = np.zeros(self.n_envs)
        _abi.check(_abi.lib().fsg_dyn_change_bladder(self._h, _abi.dptr(dv), _abi.dptr(out)),
                   dyn=True)
        return out

    # -- the robot step ----------------------------------------------------------
    def step(self, actuation, tau_ext=None, rho_fluid: float = 1000.0, g_hydro=None,
             dt: float = 0.004, substeps: int = 1, gravity=None) -> np.ndarray:
        """session.hpp:169-175 for every env; returns the per-env FSG_DYN_* flags."""
        act = np.ascontiguousarray(np.asarray(actuation, dtype=np.float64).reshape(
            self.n_envs, self.n_joints))
        te = None if tau_ext is None else np.ascontiguousarray(
            np.asarray(tau_ext, dtype=np.float64).reshape(self.n_envs, self.n_dofs))
        gh = None if g_hydro is None else np.ascontiguousarray(_v(g_hydro))
        gv = None if gravity is None else np.ascontiguousarray(_v(gravity))
        flags = np.zeros(self.n_envs, dtype=np.int32)
        _abi.check(_abi.lib().fsg_dyn_step(self._h, _abi.dptr(act), _abi.dptr(te), float(rho_fluid),
                                           _abi.dptr(gh), float(dt), int(substeps), _abi.dptr(gv),
                                           _abi.iptr(flags)), dyn=True)
        return flags

    def step_device(self, actuation, tau_ext=None, rho_fluid: float = 1000.0, g_hydro=None,
                    dt: float = 0.004, substeps: int = 1, gravity=None, flags=None) -> None:
        """The same on device tensors (torch float64 [E, nj] / [E, nd], int32 [E]);
        stream-ordered on the handle's stream, no host synchronisation."""
        gh = None if g_hydro is None else np.ascontiguousarray(_v(g_hydro))
        gv = None if gravity is None else np.ascontiguousarray(_v(gravity))
        p = lambda t: None if t is None else C.c_void_p(t.data_ptr())
        _abi.check(_abi.lib().fsg_dyn_step_device(self._h, p(actuation), p(tau_ext),
                                                  float(rho_fluid), _abi.dptr(gh), float(dt),
                                                  int(substeps), _abi.dptr(gv), p(flags)), dyn=True)

    def set_rest(self, rest_R, rest_p) -> None:
        """RestPose::of the device poses of EnvBatch.step_dynamic use (fsg_dyn_set_rest)."""
        rR = np.ascontiguousarray(np.asarray(rest_R, dtype=np.float64).reshape(-1))
        rp = np.ascontiguousarray(np.asarray(rest_p, dtype=np.float64).reshape(-1))
        _abi.check(_abi.lib().fsg_dyn_set_rest(self._h, _abi.dptr(rR), _abi.dptr(rp)), dyn=True)

    # -- probes --------------------------------------------------------------------
    def mass_matrix(self, gravity=None):
        """(mass_matrix [E, nd, nd], bias_forces [E, nd]) at the current states."""
        nd = self.n_dofs
        M = np.zeros((self.n_envs, nd, nd))
        c = np.zeros((self.n_envs, nd))
        gv = None if gravity is None else np.ascontiguousarray(_v(gravity))
        _abi.check(_abi.lib().fsg_dyn_mass_matrix(self._h, _abi.dptr(gv), _abi.dptr(M),
                                                  _abi.dptr(c)), dyn=True)
        return M, c

    def poses(self, rest_R, rest_p) -> np.ndarray:
        """[E, 30 * SKIN_MAX_LINKS] packed fsg_body_pose of every env (FK + BoneTransforms::of)."""
        rR = np.ascontiguousarray(np.asarray(rest_R, dtype=np.float64).reshape(-1))
        rp = np.ascontiguousarray(np.asarray(rest_p, dtype=np.float64).reshape(-1))
        out = np.zeros((self.n_envs, 30 * _abi.SKIN_MAX_LINKS))
        _abi.check(_abi.lib().fsg_dyn_poses(self._h, _abi.dptr(rR), _abi.dptr(rp),
                                            out.ctypes.data_as(C.c_void_p)), dyn=True)
        return out


# ------------------------------------------------------------------ koi robot --
def koi_robot(body, art, rho_body: float = 1080.0, ballast_drop: float = 0.010,
              stiffness: float = 1.0, damping: float = 0.02, torque_limit: float = 0.3,
              joint_limit: float = 0.7, bladder_capacity_factor: float = 2.5) -> Robot:
    """A dynamic koi for the synthetic scenes: the articulation of
    ``scenes.koi_articulation`` with mass properties lumped from the surface
    samples as assign_mass_properties does from the mesh (model_builder.hpp:61-101;
    FishDesign defaults, model_builder.hpp:22-41), the body volume taken as the
    elliptic tube's.  Rest pose: base at the origin, identity rotations."""
    Lb = art.n_links
    rest_p = np.zeros((Lb, 3))
    for i in range(1, Lb):
        rest_p[i] = rest_p[art.parent[i]] + art.joint_origin[i]
    A = body.areas
    a_total = float(A.sum())
    # tube volume: sum over slices of pi a b ds (the koi profile of scenes.koi_body)
    xs = np.unique(body.rest[:, 0])
    ds = body.length / len(xs)
    v_total = 0.0
    for x in xs:
        sl = body.rest[body.rest[:, 0] == x]
        v_total += math.pi * np.abs(sl[:, 1]).max() * np.abs(sl[:, 2]).max() * ds
    links = []
    for b in range(Lb):
        w = art.weights[:, b] * A
        wa = float(w.sum())
        l = Link(parent=art.parent[b], joint=FREE if b == 0 else REVOLUTE,
                 joint_origin=art.joint_origin[b].copy(), axis=art.axis[b].copy() if b else
                 np.array([0.0, 0.0, 1.0]))
        if wa <= 0.0:
            l.mass, l.inertia_com = 1e-4, 1e-8 * np.eye(3)
        else:
            com_w = (w[:, None] * body.rest).sum(0) / wa
            com_l = com_w - rest_p[b]
            l.displaced_volume = v_total * wa / a_total
            l.mass = rho_body * l.displaced_volume
            l.volume_centroid = com_l
            l.com = com_l - np.array([0.0, 0.0, ballast_drop])
            r = body.rest - com_w
            I = np.einsum("m,mij->ij", w, (r * r).sum(1)[:, None, None] * np.eye(3)[None] -
                          r[:, :, None] * r[:, None, :])
            l.inertia_com = I * (l.mass / wa) + 1e-9 * np.eye(3)
        if b:
            l.stiffness, l.damping, l.torque_limit = stiffness, damping, torque_limit
            l.limit_lo, l.limit_hi = -joint_limit, joint_limit
        links.append(l)
    robot = Robot(links)
    trim = robot.neutral_trim_volume(1000.0)
    robot.bladder = Bladder(volume=max(trim, 0.0), volume_min=0.0,
                            volume_max=bladder_capacity_factor * max(trim, 0.0) + 1e-9,
                            rate_bound=1e-6, centroid=links[0].volume_centroid.copy())
    return robot


def rest_pose(robot: Robot):
    """RestPose::of (skinning.hpp): world rotation / position of every link at
    JointState::zero -> (rest_R [L,3,3], rest_p [L,3])."""
    Lb = robot.n_links
    R = np.zeros((Lb, 3, 3))
    p = np.zeros((Lb, 3))
    R[0] = np.eye(3)
    for i in range(1, Lb):
        l = robot.links[i]
        pa = l.parent
        R[i] = R[pa] @ np.asarray(l.joint_rotation, dtype=np.float64).reshape(3, 3)
        p[i] = p[pa] + R[pa] @ _v(l.joint_origin)
    return R, p
