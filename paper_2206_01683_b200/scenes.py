"""Synthetic scenes for the BASELINE.json configurations (host-side inputs).

The reference produces marker state with its robot stack (blue-noise
sampling, sampling.hpp:164-303; linear-blend skinning, skinning.hpp:105-126;
Featherstone dynamics).  That stack is outside the hot path (SURVEY.md §2
rows 14-17), so the benchmarks drive the path with PRESCRIBED kinematics of
bodies of the same size and marker density (spacing = dx, session.hpp:33):

* ``sphere``   : icosphere-like rigid sphere, Fibonacci-sampled (C1)
* ``koi``      : koi-profile elliptic tube (model_builder.hpp:224-232,
                 meshes.hpp:108-153 geometry, 0.4 m long) with a travelling
                 body wave at the SineGait frequency (gait.hpp:13-44, 2 Hz)

Each scene yields, per step, world-frame marker points / velocities /
normals / areas and (for local-frame scenes) the FrameState the follower
would produce.  Everything is plain numpy; nothing here runs on the GPU.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from ._abi import SKIN_MAX_LINKS as SKIN_L
from .session import FrameState


@dataclass
class Body:
    rest: np.ndarray      # [m,3] body-frame rest points
    normals: np.ndarray   # [m,3] body-frame rest normals
    areas: np.ndarray     # [m]
    length: float = 0.0

    @property
    def m(self) -> int:
        return int(self.rest.shape[0])


def sphere_body(radius: float, spacing: float) -> Body:
    """Fibonacci sphere with ~ 4 pi R^2 / spacing^2 markers."""
    n = max(8, int(round(4.0 * math.pi * radius * radius / (spacing * spacing))))
    k = np.arange(n) + 0.5
    zc = 1.0 - 2.0 * k / n
    r = np.sqrt(np.maximum(0.0, 1.0 - zc * zc))
    phi = math.pi * (3.0 - math.sqrt(5.0)) * k
    nrm = np.stack([r * np.cos(phi), r * np.sin(phi), zc], axis=1)
    return Body(radius * nrm, nrm.copy(), np.full(n, 4.0 * math.pi * radius * radius / n), 2 * radius)


def koi_body(spacing: float, length: float = 0.4) -> Body:
    """Elliptic-section tube with the koi width/height profiles (model_builder.hpp:229-230)."""
    width = lambda t: 0.085 * math.sin((1.0 - t) ** 0.8 * math.pi * 0.92 + 0.05)
    height = lambda t: 0.12 * math.sin((1.0 - t) ** 0.9 * math.pi * 0.88 + 0.08)
    ns = max(4, int(round(length / spacing)))
    pts, nrms, areas = [], [], []
    ds = length / ns
    for s in range(ns):
        t = (s + 0.5) / ns
        x = 0.5 * length - t * length
        a, b = 0.5 * max(width(t), 1e-4), 0.5 * max(height(t), 1e-4)
        h = ((a - b) / (a + b)) ** 2
        perim = math.pi * (a + b) * (1 + 3 * h / (10 + math.sqrt(4 - 3 * h)))
        nt = max(6, int(round(perim / spacing)))
        ang = 2.0 * math.pi * (np.arange(nt) + 0.5 * (s % 2)) / nt
        y, z = a * np.cos(ang), b * np.sin(ang)
        ny, nz = np.cos(ang) / a, np.sin(ang) / b
        nn = np.sqrt(ny * ny + nz * nz)
        pts.append(np.stack([np.full(nt, x), y, z], axis=1))
        nrms.append(np.stack([np.zeros(nt), ny / nn, nz / nn], axis=1))
        areas.append(np.full(nt, perim * ds / nt))
    return Body(np.concatenate(pts), np.concatenate(nrms), np.concatenate(areas), length)


# ------------------------------------------------------- articulated koi --
# A skinned koi for the device-side marker refresh: a
# floating base and N_SPINE revolute z joints down the spine (koi_design's 5
# spine joints, model_builder.hpp), every marker blended between the two
# nearest bones.  Forward kinematics is the caller's (host) work in the
# reference -- dynamics.hpp:23-61, restated here with numpy to produce the
# per-link pose the path consumes; the joint angles follow a kinematic
# travelling wave at the SineGait frequency and phase step (gait.hpp:13-44).
N_SPINE = 5


@dataclass
class Articulation:
    parent: list
    dof_index: list
    axis: np.ndarray          # [L,3] normalized
    joint_origin: np.ndarray  # [L,3] in parent coordinates
    weights: np.ndarray       # [m, L]
    floating_base: bool = True

    @property
    def n_links(self) -> int:
        return len(self.parent)

    @property
    def n_dofs(self) -> int:
        return (6 if self.floating_base else 0) + sum(1 for d in self.dof_index[1:] if d >= 0)


def koi_articulation(body: Body, n_spine: int = N_SPINE) -> Articulation:
    L = body.length
    nb = n_spine + 1
    seg = L / nb
    xj = [0.5 * L - j * seg for j in range(1, nb)]  # joint j between bone j-1 and j
    origin = np.zeros((nb, 3))
    origin[1] = (xj[0], 0.0, 0.0)
    for j in range(2, nb):
        origin[j] = (xj[j - 1] - xj[j - 2], 0.0, 0.0)
    axis = np.zeros((nb, 3))
    axis[1:, 2] = 1.0
    u = (0.5 * L - body.rest[:, 0]) / seg - 0.5  # bone centres at integer u
    W = np.zeros((body.m, nb))
    k0 = np.clip(np.floor(u).astype(int), 0, nb - 1)
    f = u - k0
    for i in range(body.m):
        if u[i] <= 0.0:
            W[i, 0] = 1.0
        elif k0[i] >= nb - 1:
            W[i, nb - 1] = 1.0
        else:
            W[i, k0[i]] = 1.0 - f[i]
            W[i, k0[i] + 1] = f[i]
    return Articulation(list(range(-1, nb - 1)), [0] + [6 + j for j in range(nb - 1)], axis,
                        origin, W)


def _angle_axis(theta: float, a: np.ndarray) -> np.ndarray:
    """Eigen::AngleAxisd(theta, a).toRotationMatrix() (unit a)."""
    c, s_ = math.cos(theta), math.sin(theta)
    x, y, z = a
    C = 1.0 - c
    return np.array([[c + x * x * C, x * y * C - z * s_, x * z * C + y * s_],
                     [y * x * C + z * s_, c + y * y * C, y * z * C - x * s_],
                     [z * x * C - y * s_, z * y * C + x * s_, c + z * z * C]])


def forward_kinematics(art: Articulation, base_R, base_p, v_gen, q):
    """KinematicsCache of dynamics.hpp:23-61 (joint_rotation = identity):
    -> R_world[L,3,3], p_world[L,3], omega_world[L,3], v_origin_world[L,3]."""
    L = art.n_links
    R = np.zeros((L, 3, 3))
    p = np.zeros((L, 3))
    vb = np.zeros((L, 6))
    R[0], p[0] = base_R, base_p
    vb[0] = v_gen[:6] if art.floating_base else 0.0
    for i in range(1, L):
        pa = art.parent[i]
        d = art.dof_index[i]
        rel = _angle_axis(q[d - 6], art.axis[i]) if d >= 0 else np.eye(3)
        R[i] = R[pa] @ rel
        p[i] = p[pa] + R[pa] @ art.joint_origin[i]
        w_pa, v_pa = vb[pa, :3], vb[pa, 3:]
        w = rel.T @ w_pa
        v = rel.T @ (v_pa - np.cross(art.joint_origin[i], w_pa))  # apply_motion (spatial.hpp:21-26)
        if d >= 0:
            w = w + art.axis[i] * v_gen[d]
        vb[i, :3], vb[i, 3:] = w, v
    om = np.einsum("lij,lj->li", R, vb[:, :3])
    vo = np.einsum("lij,lj->li", R, vb[:, 3:])
    return R, p, om, vo


def pack_pose(R, p, om, vo, rest_R, rest_p) -> np.ndarray:
    """fsg_body_pose layout (30 * SKIN_MAX_LINKS doubles): BoneTransforms::of (skinning.hpp:90-99)
    + the KinematicsCache fields."""
    L = R.shape[0]
    bR = np.einsum("lij,lkj->lik", R, rest_R)        # R_world * rest.R^T
    bt = p - np.einsum("lij,lj->li", bR, rest_p)      # p_world - R_b * rest.p
    out = np.zeros(30 * SKIN_L)
    o = 0
    for a, w in ((bR, 9), (bt, 3), (R, 9), (p, 3), (vo, 3), (om, 3)):
        out[o:o + L * w] = a.reshape(-1)
        o += SKIN_L * w
    return out


def _rotz(yaw: float) -> np.ndarray:
    c, s = math.cos(yaw), math.sin(yaw)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


@dataclass
class Pose:
    """Prescribed base motion: position, velocity, yaw, yaw rate."""

    p: np.ndarray
    v: np.ndarray
    yaw: float = 0.0
    yaw_rate: float = 0.0


@dataclass
class Scene:
    name: str
    dims: tuple
    dx: float
    frame_mode: str
    bodies: list
    steps: int
    dt: float = 0.004
    rho: float = 1000.0
    nu: float = 0.00089
    motion: str = "oscillate"  # "oscillate" (rigid sphere) | "swim" (undulating koi)
    origins: list = field(default_factory=list)
    period_steps: int = 250
    amplitude: float = 0.0
    wave_amp: float = 0.08
    gait_hz: float = 2.0

    @property
    def n_cells(self) -> int:
        return int(np.prod(self.dims))

    @property
    def m(self) -> int:
        return int(sum(b.m for b in self.bodies))

    @property
    def offsets(self) -> np.ndarray:
        return np.concatenate([[0], np.cumsum([b.m for b in self.bodies])]).astype(np.int64)

    def base_pose(self, k: int, step: int) -> Pose:
        t = step * self.dt
        o = np.asarray(self.origins[k], dtype=np.float64)
        if self.motion == "oscillate":
            w = 2.0 * math.pi / (self.period_steps * self.dt)
            return Pose(o + np.array([self.amplitude * math.sin(w * t), 0.0, 0.0]),
                        np.array([self.amplitude * w * math.cos(w * t), 0.0, 0.0]))
        w = 2.0 * math.pi * self.gait_hz
        U0 = 0.05
        p = o + np.array([U0 * t - 0.2 * U0 / w * math.cos(w * t), 0.0, 0.0])
        v = np.array([U0 * (1.0 + 0.2 * math.sin(w * t)), 0.0, 0.0])
        return Pose(p, v, 0.1 * math.sin(w * t), 0.1 * w * math.cos(w * t))

    def frame(self, step: int) -> FrameState:
        """Frame that rides the tracked body (FrameFollower target, frame.hpp:90-119)."""
        if self.frame_mode == "none":
            return FrameState()
        t = step * self.dt
        w = 2.0 * math.pi * self.gait_hz
        U0 = 0.05
        o = np.asarray(self.origins[0], dtype=np.float64)
        # the critically damped follower (tau = 0.2 s, frame.hpp:70-125) passes
        # |H(i w)| = wn^2 / |wn^2 - w^2 + 2 i wn w| of the gait-frequency jitter
        wn = 5.0
        g = wn * wn / math.hypot(wn * wn - w * w, 2.0 * wn * w)
        ya, sa = 0.1 * g, 0.2 * g
        yaw = ya * math.sin(w * t)
        return FrameState(
            p=o + np.array([U0 * t - sa * U0 / w * math.cos(w * t), 0.0, 0.0]),
            pd=np.array([U0 * (1.0 + sa * math.sin(w * t)), 0.0, 0.0]),
            pdd=np.array([sa * U0 * w * math.cos(w * t), 0.0, 0.0]),
            q=np.array([math.cos(0.5 * yaw), 0.0, 0.0, math.sin(0.5 * yaw)]),
            omega=np.array([0.0, 0.0, ya * w * math.cos(w * t)]),
            alpha=np.array([0.0, 0.0, -ya * w * w * math.sin(w * t)]))

    # -- skinned bodies (device-side LBS + tau_ext) -------
    def articulations(self) -> list:
        if not hasattr(self, "_arts"):
            self._arts = [koi_articulation(b) if self.motion == "swim" else
                          Articulation([-1], [0], np.zeros((1, 3)), np.zeros((1, 3)),
                                       np.ones((b.m, 1))) for b in self.bodies]
            self._rest = []
            for a in self._arts:
                R, p, _, _ = forward_kinematics(a, np.eye(3), np.zeros(3), np.zeros(a.n_dofs),
                                                np.zeros(max(a.n_links - 1, 0)))
                self._rest.append((R, p))
        return self._arts

    def skin(self):
        """-> (body_offsets, skeleton specs, rest_points, rest_normals, weights list, areas)."""
        arts = self.articulations()
        from .session import Skeleton
        sks = [Skeleton(a.parent, a.dof_index, a.axis, a.floating_base, a.n_dofs) for a in arts]
        return (self.offsets, sks, np.concatenate([b.rest for b in self.bodies]),
                np.concatenate([b.normals for b in self.bodies]), [a.weights for a in arts],
                np.concatenate([b.areas for b in self.bodies]))

    def joint_state(self, k: int, step: int):
        """(base_R, base_p, v_gen, q) of body k: the base motion of base_pose and
        a travelling wave q_j = A_j sin(w t - j phase_step) down the spine."""
        a = self.articulations()[k]
        pose = self.base_pose(k, step)
        R0 = _rotz(pose.yaw)
        v = np.zeros(a.n_dofs)
        v[:3] = (0.0, 0.0, pose.yaw_rate)        # base omega, body coordinates
        v[3:6] = R0.T @ pose.v                   # base velocity, body coordinates
        nj = a.n_links - 1
        q = np.zeros(nj)
        w = 2.0 * math.pi * self.gait_hz
        t = step * self.dt
        for j in range(nj):
            A = 0.15 * (j + 1) / nj
            q[j] = A * math.sin(w * t - 0.8 * j)
            v[6 + j] = A * w * math.cos(w * t - 0.8 * j)
        return R0, pose.p, v, q

    def poses(self, step: int) -> np.ndarray:
        """[n_bodies, 30 * SKIN_MAX_LINKS] packed fsg_body_pose of every body at `step`."""
        arts = self.articulations()
        out = np.zeros((len(arts), 30 * SKIN_L))
        for k, a in enumerate(arts):
            R0, p0, v, q = self.joint_state(k, step)
            R, p, om, vo = forward_kinematics(a, R0, p0, v, q)
            out[k] = pack_pose(R, p, om, vo, *self._rest[k])
        return out

    def markers(self, step: int):
        """World-frame (points, velocities, normals, areas) of all bodies at `step`."""
        P, V, N, A = [], [], [], []
        t = step * self.dt
        for k, b in enumerate(self.bodies):
            pose = self.base_pose(k, step)
            x = b.rest.copy()
            v_body = np.zeros_like(x)
            if self.motion == "swim":
                # travelling body wave, amplitude growing toward the tail
                L = b.length
                s = np.clip((0.5 * L - x[:, 0]) / L, 0.0, 1.0)
                w = 2.0 * math.pi * self.gait_hz
                amp = self.wave_amp * L * s * s
                ph = w * t - 2.0 * math.pi * s
                x[:, 1] += amp * np.sin(ph)
                v_body[:, 1] = amp * w * np.cos(ph)
            R = _rotz(pose.yaw)
            xr = x @ R.T
            wz = np.array([0.0, 0.0, pose.yaw_rate])
            P.append(pose.p + xr)
            V.append(pose.v + np.cross(wz, xr) + v_body @ R.T)
            N.append(b.normals @ R.T)
            A.append(b.areas)
        return (np.ascontiguousarray(np.concatenate(P)), np.ascontiguousarray(np.concatenate(V)),
                np.ascontiguousarray(np.concatenate(N)), np.ascontiguousarray(np.concatenate(A)))


def make_scene(name: str) -> Scene:
    """BASELINE.json configs C1..C5 (SURVEY.md §8(d) synthetic inputs)."""
    name = name.lower()
    if name in ("c1", "sphere64"):
        dx = 0.01
        return Scene("c1: 64^3 fixed domain, rigid sphere, IB on", (64, 64, 64), dx, "none",
                     [sphere_body(0.125, dx)], 1000, origins=[np.zeros(3)], motion="oscillate",
                     amplitude=2 * dx, period_steps=250)
    if name in ("c2", "fish128"):
        dx = 0.008
        return Scene("c2: one koi in local accelerating frame, 128x64x64", (128, 64, 64), dx,
                     "translation_yaw", [koi_body(dx)], 1000, origins=[np.zeros(3)], motion="swim")
    if name in ("c3", "school256"):
        dx = 0.008
        return Scene("c3: two-koi schooling, 256x128x128 fixed domain", (256, 128, 128), dx, "none",
                     [koi_body(dx), koi_body(dx)], 500,
                     origins=[np.array([-0.3025, 0.0, 0.0]), np.array([0.3025, 0.0, 0.0])],
                     motion="swim")
    if name in ("c4", "slab512"):
        return Scene("c4: 512^3 fixed domain (pure LBM)", (512, 512, 512), 0.01, "none", [], 20,
                     origins=[])
    if name in ("c5", "env96"):
        dx = 0.01
        return Scene("c5: one 96x48x48 local-frame koi env", (96, 48, 48), dx, "translation_yaw",
                     [koi_body(dx)], 200, origins=[np.zeros(3)], motion="swim")
    raise ValueError(f"unknown scene {name!r}")
