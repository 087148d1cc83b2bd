"""Python mirror of the reference's hot-path API over the C ABI.

Names and argument meaning follow FishGym's C++ API so that tests read like
the reference's own Catch2 tests:

* ``SessionConfig``            <- sim::SessionConfig (session.hpp:12-24) + UnitMap (units.hpp:18-23)
* ``CoupledSession``           <- sim::CoupledSession (session.hpp:29-224), fluid half of step()
* ``CoupledSession.collide_and_stream / macroscopic / total_mass / total_momentum``
                               <- lbm::collide_and_stream etc. (solver.hpp:25-206)
* ``FrameState``               <- frame::FrameState (frame.hpp:13-43)
* ``StepStatus``               <- lbm::StepStatus (solver.hpp:13-20) / StepOutcome (backend.hpp:37-40)

Errors: invalid configuration raises ``InputError`` (reference: InputError),
instability is reported in the returned status, never raised.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._abi import check, dptr, iptr

BOUNDARY = {"periodic": 0, "open": 1}
KERNEL = {"peskin4": 0, "roma3": 1}
WALL = {"slip": 0, "noslip": 1}
FRAME = {"none": 0, "translation": 1, "translation_yaw": 2, "full": 3}
PRECISION = {"fp32": 0, "fp64": 1}


def tau_of(dx: float, dt: float, nu: float) -> float:
    """UnitMap::tau (units.hpp:25): 3 nu dt/dx^2 + 1/2."""
    return _abi.lib().fsg_tau(dx, dt, nu)


@dataclass
class SessionConfig:
    dims: tuple = (64, 64, 64)
    dx: float = 0.01
    dt: float = 0.004
    rho: float = 1000.0
    nu: float = 0.00089
    boundary: str = "open"
    kernel: str = "peskin4"
    wall: str = "slip"
    frame_mode: str = "translation_yaw"
    precision: str = "fp32"
    device: int = 0
    max_markers: int = 65536
    z_offset: int = 0
    nz_global: int = 0

    @staticmethod
    def lattice_units(dims, tau: float, **kw) -> "SessionConfig":
        """dx = dt = rho = 1 with nu chosen to hit tau (test_lattice.cpp:16-24)."""
        return SessionConfig(dims=tuple(dims), dx=1.0, dt=1.0, rho=1.0, nu=(tau - 0.5) / 3.0, **kw)

    def to_c(self) -> _abi.fsg_config:
        c = _abi.fsg_config()
        for k in range(3):
            c.dims[k] = int(self.dims[k])
        c.dx, c.dt, c.rho, c.nu = float(self.dx), float(self.dt), float(self.rho), float(self.nu)
        c.boundary = BOUNDARY[self.boundary]
        c.kernel = KERNEL[self.kernel]
        c.wall = WALL[self.wall]
        c.frame_mode = FRAME[self.frame_mode]
        c.precision = PRECISION[self.precision]
        c.device = int(self.device)
        c.max_markers = int(self.max_markers)
        c.z_offset = int(self.z_offset)
        c.nz_global = int(self.nz_global)
        return c

    @property
    def tau(self) -> float:
        return tau_of(self.dx, self.dt, self.nu)


@dataclass
class StepStatus:
    finite: bool
    min_f: float
    n_nonpositive_rho: int = 0
    out_of_bounds_markers: int = 0
    ok: bool = True

    def stable(self, negative_tolerance: float = 1e-3) -> bool:
        """solver.hpp:17-19 (plus the session's rho check, session.hpp:97)."""
        return self.finite and self.min_f > -negative_tolerance and self.n_nonpositive_rho == 0

    @classmethod
    def of(cls, s: _abi.fsg_status) -> "StepStatus":
        return cls(bool(s.finite), float(s.min_f), int(s.n_nonpositive_rho),
                   int(s.out_of_bounds_markers), bool(s.stable))


@dataclass
class FrameState:
    """frame::FrameState (frame.hpp:13-20), world frame; q = (w, x, y, z)."""

    p: np.ndarray = field(default_factory=lambda: np.zeros(3))
    pd: np.ndarray = field(default_factory=lambda: np.zeros(3))
    pdd: np.ndarray = field(default_factory=lambda: np.zeros(3))
    q: np.ndarray = field(default_factory=lambda: np.array([1.0, 0.0, 0.0, 0.0]))
    omega: np.ndarray = field(default_factory=lambda: np.zeros(3))
    alpha: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def packed(self) -> np.ndarray:
        """The 19 doubles of fsg_frame_state in field order."""
        buf = np.concatenate([np.asarray(getattr(self, n), dtype=np.float64).reshape(-1)
                              for n in ("p", "pd", "pdd", "q", "omega", "alpha")])
        if buf.size != 19:
            raise ValueError("FrameState: p, pd, pdd, omega, alpha need 3 values, q needs 4")
        return buf

    def to_c(self) -> _abi.fsg_frame_state:
        return _abi.fsg_frame_state.from_buffer_copy(self.packed())

    @classmethod
    def of(cls, c: _abi.fsg_frame_state) -> "FrameState":
        return cls(*(np.array(list(getattr(c, n))) for n in ("p", "pd", "pdd", "q", "omega", "alpha")))


class FrameFollower:
    """frame::FrameFollower (frame.hpp:70-125): critically damped tracker of
    the robot base producing the local frame's state (host code, fp64,
    bit-identical to the reference).  mode: none | translation |
    translation_yaw | full; time_constant in seconds (frame.hpp:75-76)."""

    def __init__(self, mode: str = "translation", time_constant: float = 0.2):
        if mode not in FRAME:
            raise ValueError(f"unknown frame mode '{mode}'")  # parse_follow_mode (frame.hpp:57-63)
        self.mode = mode
        h = C.c_void_p()
        check(_abi.lib().fsg_follower_create(FRAME[mode], float(time_constant), C.byref(h)))
        self._h = h

    def reset(self, p, yaw: float = 0.0) -> None:
        """Snap to a target with zero derivatives (episode reset, frame.hpp:81-87)."""
        pa = np.ascontiguousarray(p, dtype=np.float64).reshape(3)
        check(_abi.lib().fsg_follower_reset(self._h, dptr(pa), float(yaw)))

    def step(self, target_p, target_q, dt: float) -> None:
        """One filter step toward the base pose (position, quaternion w,x,y,z)."""
        tp = np.ascontiguousarray(target_p, dtype=np.float64).reshape(3)
        tq = np.ascontiguousarray(target_q, dtype=np.float64).reshape(4)
        check(_abi.lib().fsg_follower_step(self._h, dptr(tp), dptr(tq), float(dt)))

    def state(self) -> FrameState:
        c = _abi.fsg_frame_state()
        check(_abi.lib().fsg_follower_state(self._h, C.byref(c)))
        return FrameState.of(c)

    def close(self) -> None:
        if getattr(self, "_h", None):
            _abi.lib().fsg_follower_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


POSE_DOUBLES = 30 * _abi.SKIN_MAX_LINKS  # sizeof(fsg_body_pose) / 8


@dataclass
class Skeleton:
    """Topology of a robot (skeleton.hpp:16-93) as the skinning path needs it:
    parent of each link, velocity-space index of its revolute dof (-1: none)
    and the normalized joint axis (links[i].axis.normalized())."""

    parent: list
    dof_index: list
    axis: np.ndarray
    floating_base: bool = True
    n_dofs: int = 0

    @property
    def n_links(self) -> int:
        return len(self.parent)

    def to_c(self) -> _abi.fsg_skeleton:
        c = _abi.fsg_skeleton()
        c.n_links = self.n_links
        c.floating_base = 1 if self.floating_base else 0
        c.n_dofs = int(self.n_dofs)
        ax = np.asarray(self.axis, dtype=np.float64).reshape(-1, 3)
        for j in range(self.n_links):
            c.parent[j] = int(self.parent[j])
            c.dof_index[j] = int(self.dof_index[j])
            for k in range(3):
                c.axis[j][k] = float(ax[j, k])
        return c


@dataclass
class BodyPose:
    """One body's pose for a step: BoneTransforms::of (skinning.hpp:85-102)
    and the KinematicsCache fields (dynamics.hpp:14-21), per link."""

    bone_R: np.ndarray          # [L,3,3]
    bone_t: np.ndarray          # [L,3]
    R_world: np.ndarray         # [L,3,3]
    p_world: np.ndarray         # [L,3]
    v_origin_world: np.ndarray  # [L,3]
    omega_world: np.ndarray     # [L,3]

    def packed(self) -> np.ndarray:
        L = _abi.SKIN_MAX_LINKS
        out = np.zeros(POSE_DOUBLES)
        o = 0
        for a, w in ((self.bone_R, 9), (self.bone_t, 3), (self.R_world, 9), (self.p_world, 3),
                     (self.v_origin_world, 3), (self.omega_world, 3)):
            a = np.asarray(a, dtype=np.float64).reshape(-1, w)
            out[o:o + a.shape[0] * w] = a.reshape(-1)
            o += L * w
        return out


class CoupledSession:
    """One device-resident IB-LBM domain (sim::CoupledSession, session.hpp:29-224)."""

    def __init__(self, cfg: SessionConfig, _borrowed=None):
        self.cfg = cfg
        L = _abi.lib()
        if _borrowed is None:
            h = C.c_void_p()
            check(L.fsg_create(C.byref(cfg.to_c()), C.byref(h)))
        else:
            h = C.c_void_p(_borrowed)  # an env of an EnvBatch: the batch owns it
        self._owned = _borrowed is None
        self._h = h
        self._L = L
        self._fs_c = _abi.fsg_frame_state()
        self._fs_ref = C.byref(self._fs_c)
        self._fs_view = np.frombuffer(self._fs_c, dtype=np.float64)
        self._st = _abi.fsg_status()
        self._st_ref = C.byref(self._st)
        self._st_addr = C.addressof(self._st)
        self._fs_addr = C.addressof(self._fs_c)
        self.dims = tuple(int(d) for d in cfg.dims)
        self.n_cells = int(np.prod(self.dims))
        self.m = 0
        self.n_bodies = 0

    # -- lifetime --------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None):
            if getattr(self, "_owned", True):
                _abi.lib().fsg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        return _abi.lib().fsg_stream(self._h) or 0

    # -- LatticeGrid -----------------------------------------------------
    def reset_to_rest(self) -> None:
        check(_abi.lib().fsg_reset_rest(self._h))

    def initialize(self, rho: np.ndarray, u: np.ndarray) -> None:
        """LatticeGrid::initialize (lattice.hpp:107-116); rho[n], u[n,3] in cell order."""
        rho = np.ascontiguousarray(rho, dtype=np.float64).reshape(-1)
        u = np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
        assert rho.size == self.n_cells and u.size == 3 * self.n_cells
        check(_abi.lib().fsg_initialize(self._h, dptr(rho), dptr(u)))

    def set_f(self, f: np.ndarray) -> None:
        f = np.ascontiguousarray(f, dtype=np.float64).reshape(-1)
        assert f.size == 19 * self.n_cells
        check(_abi.lib().fsg_set_f(self._h, dptr(f)))

    def get_f(self) -> np.ndarray:
        """LatticeGrid::front() (post-stream state), direction-major [19*n]."""
        out = np.empty(19 * self.n_cells)
        check(_abi.lib().fsg_get_f(self._h, dptr(out)))
        return out

    # -- lbm::solver -----------------------------------------------------
    def set_force(self, F: np.ndarray | None) -> None:
        if F is None:
            check(_abi.lib().fsg_set_force(self._h, None))
            return
        F = np.ascontiguousarray(F, dtype=np.float64).reshape(-1)
        assert F.size == 3 * self.n_cells
        check(_abi.lib().fsg_set_force(self._h, dptr(F)))

    def collide_and_stream(self) -> StepStatus:
        st = _abi.fsg_status()
        check(_abi.lib().fsg_collide_and_stream(self._h, C.byref(st)))
        return StepStatus.of(st)

    def macroscopic(self):
        """lbm::macroscopic_into with the stored force -> (rho[n], u[n,3], n_nonpositive)."""
        rho = np.empty(self.n_cells)
        u = np.empty(3 * self.n_cells)
        bad = C.c_int(0)
        check(_abi.lib().fsg_macroscopic(self._h, dptr(rho), dptr(u), C.byref(bad)))
        return rho, u.reshape(-1, 3), bad.value

    def total_mass(self) -> float:
        v = C.c_double()
        check(_abi.lib().fsg_total_mass(self._h, C.byref(v)))
        return v.value

    def total_momentum(self) -> np.ndarray:
        v = np.zeros(3)
        check(_abi.lib().fsg_total_momentum(self._h, dptr(v)))
        return v

    # -- frame -----------------------------------------------------------
    def set_frame(self, fs: FrameState) -> None:
        a = self._fs_view  # per-step path: slice copies into a reused struct
        a[0:3] = fs.p
        a[3:6] = fs.pd
        a[6:9] = fs.pdd
        a[9:13] = fs.q
        a[13:16] = fs.omega
        a[16:19] = fs.alpha
        rc = self._L.fsg_set_frame(self._h, self._fs_ref)
        if rc:
            check(rc)

    def frame_state(self) -> FrameState:
        c = _abi.fsg_frame_state()
        check(_abi.lib().fsg_get_frame(self._h, C.byref(c)))
        return FrameState.of(c)

    def recenter(self, shift) -> None:
        sh = np.ascontiguousarray(np.asarray(shift, dtype=np.int32))
        check(_abi.lib().fsg_recenter(self._h, iptr(sh)))

    # -- coupled step ------------------------------------------------------
    def set_markers(self, body_offsets, points, velocities, normals, areas) -> None:
        """Per-step marker state (world frame, SI), copied into a pinned slot."""
        off = np.ascontiguousarray(body_offsets, dtype=np.int64)
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (points, velocities, normals, areas)]
        nb = len(off) - 1
        rc = self._L.fsg_set_markers(self._h, nb, off.ctypes.data, *(a.ctypes.data for a in arrs))
        if rc:
            check(rc)
        self.m = int(off[-1]) if nb > 0 else 0
        self.n_bodies = nb

    def set_markers_device(self, body_offsets, d_points: int, d_velocities: int, d_normals: int,
                           d_areas: int) -> None:
        off = np.ascontiguousarray(np.asarray(body_offsets, dtype=np.int64))
        nb = len(off) - 1
        check(_abi.lib().fsg_set_markers_device(self._h, nb, off.ctypes.data_as(_abi._i64p),
                                                d_points, d_velocities, d_normals, d_areas))
        self.m = int(off[-1]) if nb > 0 else 0
        self.n_bodies = nb

    # -- skinned bodies on the device -------------------
    def set_skin(self, body_offsets, skeletons, rest_points, rest_normals, weights, areas) -> None:
        """Register skinned bodies (SurfaceSamples of each robot, sampling.hpp):
        every later step refreshes the markers on the device from the pose
        (update_samples, sampling.hpp:307-322) and reduces tau_ext and the
        CouplingStats there (session.hpp:129-143).  weights: per body an
        [m_b, n_links_b] array (or all of them concatenated, flattened)."""
        off = np.ascontiguousarray(body_offsets, dtype=np.int64)
        nb = len(off) - 1
        sk = (_abi.fsg_skeleton * max(nb, 1))()
        for b, k in enumerate(skeletons):
            sk[b] = k.to_c()
        if isinstance(weights, (list, tuple)):
            weights = np.concatenate([np.asarray(w, dtype=np.float64).reshape(-1) for w in weights])
        arrs = [np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
                for a in (rest_points, rest_normals, weights, areas)]
        check(self._L.fsg_set_skin(self._h, nb, off.ctypes.data_as(_abi._i64p), sk,
                                   *(dptr(a) for a in arrs)))
        self.m = int(off[-1])
        self.n_bodies = nb
        self._ndofs = [int(k.n_dofs) for k in skeletons]
        self._nt = sum(self._ndofs)
        self._wbuf = np.empty(self._nt + 7 * nb)  # readback staging (pointer cached)
        self._wptr = self._wbuf.ctypes.data
        ends = np.cumsum(self._ndofs).tolist()
        self._tau_ranges = list(zip([0] + ends[:-1], ends))
        self._pose = (_abi.fsg_body_pose * nb)()
        self._pose_np = np.frombuffer(self._pose, dtype=np.float64).reshape(nb, POSE_DOUBLES)
        self._pose_addr = C.addressof(self._pose)

    def set_pose(self, poses) -> None:
        """This step's pose of every skinned body: a list of BodyPose, or an
        [n_bodies, POSE_DOUBLES] array already packed in fsg_body_pose order."""
        if getattr(self, "_pose", None) is None:  # no skinned bodies: the ABI reports it
            check(self._L.fsg_set_pose(self._h, None))
        if isinstance(poses, np.ndarray):
            self._pose_np[...] = poses.reshape(self._pose_np.shape)
        else:
            for b, p in enumerate(poses):
                self._pose_np[b] = p.packed()
        rc = self._L.fsg_set_pose(self._h, self._pose)
        if rc:
            check(rc)

    def body_wrench(self):
        """-> (tau_ext per body [list of n_dofs arrays], stats[n_bodies, 7]) of the last step."""
        rc = self._L.fsg_get_body_wrench(self._h, self._wptr, self._wptr + 8 * self._nt)
        if rc:
            check(rc)
        buf = self._wbuf.copy()
        return [buf[a:b] for a, b in self._tau_ranges], buf[self._nt:].reshape(-1, 7)

    def step_skinned(self, frame, poses):
        """The robot loop's per-step exchange in one ABI call (fsg_step_skinned):
        frame (FrameState, a packed [19] array, or None to keep it), poses
        ([n_bodies, POSE_DOUBLES] packed or a list of BodyPose) -> (StepStatus,
        tau_ext per body, stats[n_bodies, 7])."""
        fp = None
        if frame is not None:
            self._fs_view[:] = frame if isinstance(frame, np.ndarray) else frame.packed()
            fp = self._fs_addr
        if isinstance(poses, np.ndarray):
            self._pose_np[...] = poses.reshape(self._pose_np.shape)
        else:
            for b, p in enumerate(poses):
                self._pose_np[b] = p.packed()
        rc = self._L.fsg_step_skinned(self._h, fp, self._pose_addr, self._st_addr, self._wptr,
                                      self._wptr + 8 * self._nt)
        if rc:
            check(rc)
        buf = self._wbuf.copy()
        return (StepStatus.of(self._st), [buf[a:b] for a, b in self._tau_ranges],
                buf[self._nt:].reshape(-1, 7))

    def markers(self):
        """-> (points, velocities, normals) [m, 3] the last step used."""
        a = [np.empty(3 * self.m) for _ in range(3)]
        check(self._L.fsg_get_markers(self._h, *(dptr(x) for x in a)))
        return tuple(x.reshape(-1, 3) for x in a)

    # -- output formats --------------------------------
    def snapshot_begin(self) -> None:
        """Start an asynchronous copy of the last step's bare macro fields
        (later steps proceed while it travels)."""
        check(self._L.fsg_snapshot_begin(self._h))

    def snapshot_wait(self):
        """-> (rho[n], u[n,3]) of the last snapshot (lattice units)."""
        n = int(np.prod(self.cfg.dims))
        rho, u = np.empty(n), np.empty(3 * n)
        check(self._L.fsg_snapshot_wait(self._h, dptr(rho), dptr(u)))
        return rho, u.reshape(-1, 3)

    def write_vtk(self, path: str, origin=(0.0, 0.0, 0.0)) -> None:
        """lbm::write_vtk (vtk.hpp:15-38) of the last snapshot."""
        o = np.ascontiguousarray(origin, dtype=np.float64)
        check(self._L.fsg_write_vtk(self._h, os.fsencode(path), dptr(o)))

    def step(self) -> StepStatus:
        """Fluid half of CoupledSession::step (session.hpp:94-166)."""
        st = self._st
        rc = self._L.fsg_step(self._h, self._st_ref)
        if rc:
            check(rc)
        return StepStatus.of(st)

    def step_async(self) -> None:
        rc = self._L.fsg_step_async(self._h)
        if rc:
            check(rc)

    def last_status(self) -> StepStatus:
        st = self._st
        rc = self._L.fsg_last_status(self._h, self._st_ref)
        if rc:
            check(rc)
        return StepStatus.of(st)

    def marker_forces(self):
        """-> (force_world[m,3] on the fluid, valid[m], stats[n_bodies,7])."""
        fw = np.empty(3 * self.m)
        valid = np.empty(self.m, dtype=np.int32)
        stats = np.zeros(7 * max(self.n_bodies, 1))
        rc = self._L.fsg_get_marker_forces(self._h, fw.ctypes.data, valid.ctypes.data,
                                           stats.ctypes.data)
        if rc:
            check(rc)
        return fw.reshape(-1, 3), valid, stats[: 7 * self.n_bodies].reshape(-1, 7)

    def macro(self):
        """CoupledSession::macro() after step(): bare (rho[n], u[n,3])."""
        rho = np.empty(self.n_cells)
        u = np.empty(3 * self.n_cells)
        check(_abi.lib().fsg_get_macro(self._h, dptr(rho), dptr(u)))
        return rho, u.reshape(-1, 3)

    def set_force_capture(self, on: bool = True) -> None:
        """fp32 coupled steps: make force() return the body force the collision
        kernel consumed (captured cell by cell) instead of a rebuild."""
        check(_abi.lib().fsg_set_force_capture(self._h, 1 if on else 0))

    def force(self) -> np.ndarray:
        """BodyForceField of the last step (IB + virtual force), [n,3]."""
        F = np.empty(3 * self.n_cells)
        check(_abi.lib().fsg_get_force(self._h, dptr(F)))
        return F.reshape(-1, 3)

    def stencils(self) -> np.ndarray:
        """Integer stencil ranges of the last step: [m, 6] = lo(x,y,z), hi(x,y,z)."""
        out = np.zeros(6 * self.m, dtype=np.int32)
        check(_abi.lib().fsg_get_stencils(self._h, iptr(out)))
        return out.reshape(-1, 6)

    # -- measurement -----------------------------------------------------------
    def profile(self, enable: bool = True) -> None:
        """Bracket every step's kernels with CUDA events on the session stream."""
        check(_abi.lib().fsg_profile_enable(self._h, 1 if enable else 0))

    def profile_read(self):
        """-> (device ms of the timed steps, timed steps) accumulated since enable/read."""
        a = C.c_double()
        n = C.c_int()
        check(_abi.lib().fsg_profile_read(self._h, C.byref(a), C.byref(n)))
        return a.value, n.value

    # -- z-slab halos ----------------------------------------------------------
    def halo_bytes(self) -> int:
        return int(_abi.lib().fsg_halo_bytes(self._h))

    def halo_pack(self, d_send_lo: int, d_send_hi: int) -> None:
        check(_abi.lib().fsg_halo_pack(self._h, d_send_lo, d_send_hi))

    def halo_unpack(self, d_recv_lo: int | None, d_recv_hi: int | None) -> None:
        check(_abi.lib().fsg_halo_unpack(self._h, d_recv_lo, d_recv_hi))

    def halo_buffers(self):
        """-> device pointers (send_lo, send_hi, recv_lo, recv_hi), halo_bytes() each."""
        p = [C.c_void_p() for _ in range(4)]
        check(_abi.lib().fsg_halo_buffers(self._h, *(C.byref(x) for x in p)))
        return tuple(int(x.value or 0) for x in p)

    def halo_begin(self, comm_stream: int) -> None:
        """comm_stream waits until this step's boundary planes are packed."""
        check(_abi.lib().fsg_halo_begin(self._h, comm_stream))

    def halo_end(self, comm_stream: int, have_lo: bool, have_hi: bool) -> None:
        """The session waits for comm_stream, then unpacks the received planes."""
        check(_abi.lib().fsg_halo_end(self._h, comm_stream, int(have_lo), int(have_hi)))

    # -- z-slab peer transport (fsg_peer_*: the halo exchange inside the library)
    def peer_export(self) -> bytes:
        """This slab's peer handle (FSG_PEER_HANDLE_BYTES bytes: CUDA IPC handles
        of its buffers and delivery counters, its geometry)."""
        buf = C.create_string_buffer(_abi.PEER_HANDLE_BYTES)
        check(_abi.lib().fsg_peer_export(self._h, buf))
        return buf.raw

    def peer_connect(self, lower: bytes | None, upper: bytes | None) -> None:
        """Connect to the neighbours' handles (None at a closed global face);
        from then on step_async() runs the whole sharded step."""
        check(_abi.lib().fsg_peer_connect(self._h, lower, upper))

    def peer_disconnect(self) -> None:
        check(_abi.lib().fsg_peer_disconnect(self._h))


class EnvBatch:
    """n_envs independent env sessions of one fp32 configuration stepped
    together by one marker launch and one collide/stream launch
    (fsg_batch_*; BASELINE config 5).  ``envs[e]`` is an ordinary
    CoupledSession: set its frame and markers, read its status, forces and
    fields as usual; the batch owns it."""

    def __init__(self, cfg: SessionConfig, n_envs: int):
        L = _abi.lib()
        h = C.c_void_p()
        check(L.fsg_batch_create(C.byref(cfg.to_c()), int(n_envs), C.byref(h)))
        self._h, self._L = h, L
        self.cfg = cfg
        self.envs = [CoupledSession(cfg, _borrowed=L.fsg_batch_session(h, e)) for e in range(n_envs)]

    def step_async(self) -> None:
        rc = self._L.fsg_batch_step_async(self._h)
        if rc:
            check(rc)

    def step(self) -> list:
        """One coupled step of every env -> per-env StepStatus."""
        sts = (_abi.fsg_status * len(self.envs))()
        check(self._L.fsg_batch_step(self._h, sts))
        return [StepStatus.of(x) for x in sts]

    def step_skinned(self, frames, poses):
        """Every env skinned (set_skin on each): frames ([E, 19] packed, a list
        of FrameState, or None to keep) and poses ([E, POSE_DOUBLES] packed) in, one
        batched step -> (statuses, tau_ext per env, stats[E, 7])."""
        E = len(self.envs)
        if not hasattr(self, "_bpose"):
            self._bpose = (_abi.fsg_body_pose * E)()
            self._bpose_np = np.frombuffer(self._bpose, dtype=np.float64).reshape(E, POSE_DOUBLES)
            self._bframe = (_abi.fsg_frame_state * E)()
            self._bframe_np = np.frombuffer(self._bframe, dtype=np.float64).reshape(E, 19)
            self._bst = (_abi.fsg_status * E)()
            self._bnd = [getattr(s, "_nt", 0) for s in self.envs]
            self._bw = np.empty(sum(self._bnd) + 7 * E)
        fp = None
        if frames is not None:
            if isinstance(frames, np.ndarray):
                self._bframe_np[...] = frames.reshape(E, 19)
            else:
                for e, f in enumerate(frames):
                    self._bframe_np[e] = f.packed()
            fp = C.addressof(self._bframe)
        self._bpose_np[...] = np.asarray(poses, dtype=np.float64).reshape(E, POSE_DOUBLES)
        nt = sum(self._bnd)
        w = self._bw
        check(self._L.fsg_batch_step_skinned(self._h, fp, C.addressof(self._bpose),
                                             C.addressof(self._bst), w.ctypes.data,
                                             w.ctypes.data + 8 * nt))
        out = w.copy()
        taus, k = [], 0
        for n in self._bnd:
            taus.append(out[k:k + n])
            k += n
        return [StepStatus.of(x) for x in self._bst], taus, out[nt:].reshape(E, 7)

    def set_follow(self, time_constant: float = 0.2, recenter_threshold_cells: float = 2.0) -> None:
        """FrameFollower + recentring inside step_dynamic (session.hpp:177-195),
        in the config's frame mode; time_constant <= 0 turns it off."""
        check(self._L.fsg_batch_set_follow(self._h, float(time_constant),
                                           float(recenter_threshold_cells)))

    def center_frames(self, robots) -> None:
        """center_frame_on_robot of every env (session.hpp:210-221)."""
        check(self._L.fsg_batch_center_frames(self._h, robots._h))

    def last_shifts(self) -> np.ndarray:
        """[E, 3] recentre shifts the last step_dynamic applied."""
        out = np.zeros(3 * len(self.envs), dtype=np.int32)
        check(self._L.fsg_batch_last_shifts(self._h, out.ctypes.data))
        return out.reshape(-1, 3)

    def step_dynamic(self, robots, actuation, frames=None, rho_fluid: float | None = None,
                     g_hydro=(0.0, 0.0, -9.81), dt: float | None = None, substeps: int = 4):
        """The whole coupled step with the robots on the device
        (fsg_batch_step_dynamic): ``robots`` is a dynamics.RobotBatch with one
        robot per env (rest pose set), ``actuation`` [E, n_joints]; dt and
        rho_fluid default to (and must equal) the config's -> (statuses,
        robot flags [E], post-step states as packed fsg_joint_state rows
        [E, 55]: base_pos 3, base_quat 4, q 12, v 18, qdd 18;
        dynamics.unpack_states turns them into JointStates)."""
        E = len(self.envs)
        if not hasattr(self, "_dst"):
            self._dst = (_abi.fsg_joint_state * E)()
            self._dst_np = np.frombuffer(self._dst, dtype=np.float64).reshape(E, -1)
            self._dfl = np.zeros(E, dtype=np.int32)
            self._dst_s = (_abi.fsg_status * E)()
            self._dframe = (_abi.fsg_frame_state * E)()
            self._dframe_np = np.frombuffer(self._dframe, dtype=np.float64).reshape(E, 19)
        fp = None
        if frames is not None:
            if isinstance(frames, np.ndarray):
                self._dframe_np[...] = frames.reshape(E, 19)
            else:
                for e, f in enumerate(frames):
                    self._dframe_np[e] = f.packed()
            fp = C.addressof(self._dframe)
        act = np.ascontiguousarray(np.asarray(actuation, dtype=np.float64).reshape(-1))
        if act.size != robots.n_envs * robots.n_joints:
            raise _abi.InputError(_abi.FSG_EINPUT, f"actuation has {act.size} entries, expected "
                                                   f"{robots.n_envs} x {robots.n_joints}")
        gh = None if g_hydro is None else np.ascontiguousarray(np.asarray(g_hydro, dtype=np.float64))
        rho_fluid = self.cfg.rho if rho_fluid is None else rho_fluid
        dt = self.cfg.dt if dt is None else dt
        check(self._L.fsg_batch_step_dynamic(self._h, robots._h, fp, dptr(act), float(rho_fluid),
                                             dptr(gh), float(dt), int(substeps),
                                             C.addressof(self._dst_s), self._dfl.ctypes.data,
                                             C.addressof(self._dst)))
        return [StepStatus.of(x) for x in self._dst_s], self._dfl.copy(), self._dst_np.copy()

    def close(self) -> None:
        if getattr(self, "_h", None):
            for s in self.envs:
                s.close()
            self._L.fsg_batch_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DragBatch:
    """The empirical-drag backend's per-step surface work for n_envs robots
    on the device (fsg_drag_*; EmpiricalBackend::step, empirical.hpp:74-100,
    up to the robot integration): skinning, surface_force, tau_ext and the
    CouplingStats of every env in one launch."""

    def __init__(self, n_envs: int, k: float = 40.0, precision: str = "fp32", device: int = 0):
        L = _abi.lib()
        h = C.c_void_p()
        prec = {"fp32": 0, "fp64": 1}[precision]  # FSG_PRECISION_*
        _abi.check(L.fsg_drag_create(int(n_envs), float(k), prec, int(device), C.byref(h)), drag=True)
        self._h, self._L, self.n_envs = h, L, int(n_envs)
        self._ndofs = [0] * self.n_envs
        self._poses = (_abi.fsg_body_pose * self.n_envs)()
        self._pose_np = np.frombuffer(self._poses, dtype=np.float64).reshape(self.n_envs, POSE_DOUBLES)

    def set_skin(self, env: int, skeleton: "Skeleton", rest_points, rest_normals, weights, areas):
        arrs = [np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
                for a in (rest_points, rest_normals, weights, areas)]
        m = arrs[3].shape[0]
        sk = skeleton.to_c()
        _abi.check(self._L.fsg_drag_set_skin(self._h, int(env), C.byref(sk), m,
                                             *(dptr(a) for a in arrs)), drag=True)
        self._ndofs[env] = int(skeleton.n_dofs)

    def set_pose(self, env: int, pose) -> None:
        """pose: a BodyPose or a packed [POSE_DOUBLES] array (fsg_body_pose order)."""
        self._pose_np[env] = pose if isinstance(pose, np.ndarray) else pose.packed()
        addr = C.addressof(self._poses) + env * C.sizeof(_abi.fsg_body_pose)
        _abi.check(self._L.fsg_drag_set_pose(self._h, int(env), addr), drag=True)

    def set_poses(self, poses: np.ndarray) -> None:
        """Every env's pose: [n_envs, POSE_DOUBLES] packed fsg_body_pose rows."""
        self._pose_np[...] = np.asarray(poses, dtype=np.float64).reshape(self._pose_np.shape)
        _abi.check(self._L.fsg_drag_set_poses(self._h, C.addressof(self._poses)), drag=True)

    def step(self):
        """-> (tau_ext per env [list], stats[n_envs, 7])."""
        nt = sum(self._ndofs)
        tau = np.empty(max(nt, 1))
        stats = np.empty(7 * self.n_envs)
        _abi.check(self._L.fsg_drag_step(self._h, dptr(tau), dptr(stats)), drag=True)
        out, k = [], 0
        for n in self._ndofs:
            out.append(tau[k:k + n].copy())
            k += n
        return out, stats.reshape(-1, 7)

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._L.fsg_drag_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def format_full(v: float) -> str:
    """format_full (csv.hpp:18-22): %.17g, round-trips to the same double."""
    buf = C.create_string_buffer(40)
    _abi.check(_abi.lib().fsg_format_full(float(v), buf, 40), io=True)
    return buf.value.decode()


def write_vtk_fields(path: str, dims, rho, u, dx: float, dt: float, rho_phys: float,
                     origin=(0.0, 0.0, 0.0)) -> None:
    """lbm::write_vtk (vtk.hpp:15-38) of given lattice-unit fields."""
    d = np.ascontiguousarray(dims, dtype=np.int32)
    r = np.ascontiguousarray(rho, dtype=np.float64).reshape(-1)
    uu = np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
    o = np.ascontiguousarray(origin, dtype=np.float64)
    _abi.check(_abi.lib().fsg_write_vtk_fields(os.fsencode(path), iptr(d), dptr(r), dptr(uu), dx, dt,
                                               rho_phys, dptr(o)), io=True)


class CsvWriter:
    """CsvWriter (csv.hpp:27-66): header on construction, every row flushed
    (a truncated file is a valid prefix), %.17g values."""

    def __init__(self, path: str, columns):
        self._L = _abi.lib()
        names = (C.c_char_p * len(columns))(*(c.encode() for c in columns))
        h = C.c_void_p()
        _abi.check(self._L.fsg_csv_open(os.fsencode(path), len(columns), names, C.byref(h)), io=True)
        self._h, self.path = h, path

    def write_row(self, values) -> None:
        v = np.ascontiguousarray(values, dtype=np.float64)
        _abi.check(self._L.fsg_csv_write_row(self._h, int(v.size), dptr(v)), io=True)

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._L.fsg_csv_close(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
