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
