"""ctypes bindings for the oracle -- TEST INFRASTRUCTURE ONLY.

Two CPU libraries live here:

* ``liboracle.so``       -- the plain-C fp64 restatement (fsg_oracle.c);
* ``_ref/libfishref.so`` -- the reference's own headers compiled unmodified
                            (ref_driver.cpp), present when /root/reference was
                            available at build time (built here, shipped to
                            the GPU box as a prebuilt .so).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module.  The product package (paper_2206_01683_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfishref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_i64p = C.POINTER(C.c_int64)


def build() -> None:
    """Build liboracle.so (and _ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def iptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_ip)


def i64ptr(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_i64p)


def d3(v) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1))


def dims_arr(dims) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(dims, dtype=np.int32))


# --------------------------------------------------------------------------
class FrameState(C.Structure):
    """orc_frame_state (frame.hpp:13-20): world-frame p, pd, pdd, q(w,x,y,z), omega, alpha."""

    _fields_ = [("p", C.c_double * 3), ("pd", C.c_double * 3), ("pdd", C.c_double * 3),
                ("q", C.c_double * 4), ("omega", C.c_double * 3), ("alpha", C.c_double * 3)]

    @classmethod
    def make(cls, p=(0, 0, 0), pd=(0, 0, 0), pdd=(0, 0, 0), q=(1, 0, 0, 0), omega=(0, 0, 0),
             alpha=(0, 0, 0)):
        fs = cls()
        for name, v in (("p", p), ("pd", pd), ("pdd", pdd), ("q", q), ("omega", omega),
                        ("alpha", alpha)):
            arr = getattr(fs, name)
            for k, x in enumerate(v):
                arr[k] = float(x)
        return fs

    def as_arrays(self):
        return {k: np.array(list(getattr(self, k))) for k in ("p", "pd", "pdd", "q", "omega", "alpha")}


class FrameConsts(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("a0", C.c_double * 3), ("omega_f", C.c_double * 3),
                ("alpha_f", C.c_double * 3)]


class OrcSkeleton(C.Structure):
    """orc_skeleton (same layout as fsg_skeleton)."""

    _fields_ = [("n_links", C.c_int), ("floating_base", C.c_int), ("n_dofs", C.c_int),
                ("parent", C.c_int * 12), ("dof_index", C.c_int * 12), ("axis", (C.c_double * 3) * 12)]

    @classmethod
    def of(cls, sk):
        """From any object with parent, dof_index, axis, floating_base, n_dofs."""
        c = cls()
        c.n_links = len(sk.parent)
        c.floating_base = 1 if sk.floating_base else 0
        c.n_dofs = int(sk.n_dofs)
        ax = np.asarray(sk.axis, dtype=np.float64).reshape(-1, 3)
        for j in range(len(sk.parent)):
            c.parent[j] = int(sk.parent[j])
            c.dof_index[j] = int(sk.dof_index[j])
            for k in range(3):
                c.axis[j][k] = float(ax[j, k])
        return c


def skin_update(sk, pose_packed, rest, nrest, weights):
    """update_samples restated (sampling.hpp:307-322) -> (pts, vel, nrm) [m,3]."""
    O = oracle()
    m = int(np.asarray(rest).reshape(-1, 3).shape[0])
    out = [np.empty(3 * m) for _ in range(3)]
    O.orc_update_samples(OrcSkeleton.of(sk), dptr(d3(pose_packed)), m, dptr(d3(rest)), dptr(d3(nrest)),
                         dptr(d3(weights)), *(dptr(a) for a in out))
    return tuple(a.reshape(-1, 3) for a in out)


def skin_tau(sk, pose_packed, rest, weights, fworld, valid, vel):
    """session.hpp:129-143 for one body -> (tau[n_dofs], stats[7])."""
    O = oracle()
    m = int(np.asarray(rest).reshape(-1, 3).shape[0])
    tau = np.empty(max(int(sk.n_dofs), 1))
    stats = np.empty(7)
    O.orc_skin_tau(OrcSkeleton.of(sk), dptr(d3(pose_packed)), m, dptr(d3(rest)), dptr(d3(weights)),
                   dptr(d3(fworld)), iptr(np.ascontiguousarray(valid, dtype=np.int32)), dptr(d3(vel)),
                   dptr(tau), dptr(stats))
    return tau[: int(sk.n_dofs)], stats


def empirical_step(sk, pose_packed, rest, nrest, weights, areas, k):
    """EmpiricalBackend::step surface work restated -> (tau[n_dofs], stats[7])."""
    O = oracle()
    m = int(np.asarray(rest).reshape(-1, 3).shape[0])
    tau = np.empty(max(int(sk.n_dofs), 1))
    stats = np.empty(7)
    O.orc_empirical_step(OrcSkeleton.of(sk), dptr(d3(pose_packed)), m, dptr(d3(rest)), dptr(d3(nrest)),
                         dptr(d3(weights)), dptr(d3(areas)), float(k), dptr(tau), dptr(stats))
    return tau[: int(sk.n_dofs)], stats


_oracle = None
_ref = None


def oracle() -> C.CDLL:
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        lib = C.CDLL(ORACLE_SO)
        sig = {
            "orc_tau": (C.c_double, [C.c_double, C.c_double, C.c_double]),
            "orc_equilibrium_dir": (C.c_double, [C.c_int, C.c_double, _dp]),
            "orc_initialize": (None, [_ip, _dp, _dp, _dp]),
            "orc_macroscopic": (C.c_int, [_ip, _dp, _dp, _dp, _dp]),
            "orc_apply_open_boundary": (None, [_ip, _dp]),
            "orc_collide_and_stream": (None, [_ip, C.c_int, C.c_double, _dp, _dp, _dp, _ip, _dp]),
            "orc_total_mass": (C.c_double, [_ip, _dp]),
            "orc_total_momentum": (None, [_ip, _dp, _dp]),
            "orc_phi": (C.c_double, [C.c_int, C.c_double]),
            "orc_range": (None, [C.c_int, C.c_double, _ip, _ip]),
            "orc_marker_in_bounds": (C.c_int, [C.c_int, _ip, _dp]),
            "orc_interpolate": (None, [C.c_int, _ip, _dp, _dp, _dp]),
            "orc_spread": (None, [C.c_int, _ip, _dp, _dp, _dp]),
            "orc_direct_forcing": (None, [_dp, _dp, _dp, C.c_double, C.c_double, C.c_double,
                                          C.c_double, C.c_int, _dp]),
            "orc_frame_consts_of": (None, [C.POINTER(FrameState), C.POINTER(FrameConsts)]),
            "orc_virtual_force": (None, [C.POINTER(FrameConsts), _dp, _dp, _dp]),
            "orc_recenter": (None, [_ip, C.c_double, _dp, _dp, _ip, C.POINTER(FrameState)]),
            "orc_session_create": (C.c_void_p, [_ip, C.c_double, C.c_double, C.c_double, C.c_double,
                                                C.c_int, C.c_int, C.c_int, C.c_int]),
            "orc_session_destroy": (None, [C.c_void_p]),
            "orc_session_f": (_dp, [C.c_void_p]),
            "orc_session_force": (_dp, [C.c_void_p]),
            "orc_session_rho": (_dp, [C.c_void_p]),
            "orc_session_u": (_dp, [C.c_void_p]),
            "orc_session_set_frame": (None, [C.c_void_p, C.POINTER(FrameState)]),
            "orc_session_get_frame": (None, [C.c_void_p, C.POINTER(FrameState)]),
            "orc_session_step": (C.c_int, [C.c_void_p, C.c_int, _i64p, _dp, _dp, _dp, _dp, _dp,
                                           _ip, _dp, _ip, _dp]),
            "orc_session_recenter": (None, [C.c_void_p, _ip]),
            "orc_update_samples": (None, [C.POINTER(OrcSkeleton), _dp, C.c_int, _dp, _dp, _dp,
                                          _dp, _dp, _dp]),
            "orc_skin_tau": (None, [C.POINTER(OrcSkeleton), _dp, C.c_int, _dp, _dp, _dp, _ip,
                                    _dp, _dp, _dp]),
            "orc_empirical_step": (None, [C.POINTER(OrcSkeleton), _dp, C.c_int, _dp, _dp, _dp, _dp,
                                          C.c_double, _dp, _dp]),
            "orc_quat_exp": (None, [_dp, _dp]),
            "orc_quat_to_R": (None, [_dp, _dp]),
            "orc_forward_kinematics": (None, [C.c_void_p, C.c_void_p, C.c_void_p]),
            "orc_mass_matrix": (None, [C.c_void_p, C.c_void_p, _dp]),
            "orc_bias_forces": (None, [C.c_void_p, C.c_void_p, C.c_void_p, _dp, _dp]),
            "orc_internal_forces": (C.c_int, [C.c_void_p, C.c_void_p, _dp, _dp]),
            "orc_joint_limit_forces": (None, [C.c_void_p, C.c_void_p, _dp]),
            "orc_llt_solve": (C.c_int, [C.c_int, _dp, _dp, _dp]),
            "orc_forward_dynamics": (C.c_int, [C.c_void_p, C.c_void_p, _dp, _dp, _dp, _dp]),
            "orc_buoyancy_gravity_forces": (None, [C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                                                   _dp, _dp]),
            "orc_integrate": (C.c_int, [C.c_void_p, C.c_void_p, _dp, _dp, C.c_double, C.c_int, _dp]),
            "orc_robot_step": (C.c_int, [C.c_void_p, C.c_void_p, C.c_double, _dp, _dp, C.c_double,
                                         _dp, C.c_double, C.c_int, _dp]),
            "orc_mechanical_energy": (C.c_double, [C.c_void_p, C.c_void_p, _dp]),
            "orc_dyn_pose": (None, [C.c_void_p, C.c_void_p, _dp, _dp, C.c_void_p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _oracle = lib
    return _oracle


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        vp = C.c_void_p
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_write_vtk": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_double,
                                        C.c_double, C.c_double, C.c_double, _dp]),
            "ref_csv_write": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_char_p), C.c_int, _dp]),
            "ref_csv_read": (C.c_int, [C.c_char_p, C.c_int, _dp, _ip]),
            "ref_units_tau": (C.c_double, [C.c_double] * 4),
            "ref_units_validate": (C.c_int, [C.c_double] * 4),
            "ref_rng_uniform": (None, [C.c_uint64, C.c_int64, _dp]),
            "ref_rng_normal": (None, [C.c_uint64, C.c_int64, _dp]),
            "ref_session_create": (vp, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                        C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int]),
            "ref_session_destroy": (None, [vp]),
            "ref_n_cells": (C.c_int64, [vp]),
            "ref_reset_rest": (None, [vp]),
            "ref_set_f": (None, [vp, _dp]),
            "ref_get_f": (None, [vp, _dp]),
            "ref_initialize": (None, [vp, _dp, _dp]),
            "ref_set_force": (None, [vp, _dp]),
            "ref_get_force": (None, [vp, _dp]),
            "ref_collide_and_stream": (None, [vp, _ip, _dp]),
            "ref_apply_open_boundary": (None, [vp]),
            "ref_macroscopic": (C.c_int, [vp, _dp, _dp]),
            "ref_total_mass": (C.c_double, [vp]),
            "ref_total_momentum": (None, [vp, _dp]),
            "ref_kinetic_energy": (C.c_double, [vp]),
            "ref_set_frame": (None, [vp, _dp, _dp, _dp, _dp, _dp, _dp]),
            "ref_get_frame_p": (None, [vp, _dp]),
            "ref_frame_rotation": (None, [vp, _dp]),
            "ref_recenter": (None, [vp, _ip]),
            "ref_session_step": (C.c_int, [vp, C.c_int, _i64p, _dp, _dp, _dp, _dp, _dp, _ip, _dp,
                                           _ip, _dp]),
            "ref_get_macro": (None, [vp, _dp, _dp]),
            "ref_session_marker_xlat": (None, [vp, C.c_int64, _dp, _dp]),
            "ref_phi": (C.c_double, [C.c_int, C.c_double]),
            "ref_range": (None, [C.c_int, C.c_double, _ip, _ip]),
            "ref_marker_in_bounds": (C.c_int, [C.c_int, _ip, _dp]),
            "ref_interpolate": (None, [C.c_int, _ip, _dp, C.c_int, _dp, _dp]),
            "ref_spread": (None, [C.c_int, _ip, C.c_int, _dp, _dp, _dp]),
            "ref_direct_forcing": (None, [_dp, _dp, _dp, C.c_double, C.c_double, C.c_double,
                                          C.c_double, C.c_int, _dp]),
            "ref_virtual_force": (None, [_dp, _dp, _dp, _dp, _dp, _dp, _dp]),
            "ref_follower_create": (vp, [C.c_int, C.c_double]),
            "ref_follower_destroy": (None, [vp]),
            "ref_follower_reset": (None, [vp, _dp, C.c_double]),
            "ref_follower_step": (None, [vp, _dp, _dp, C.c_double]),
            "ref_follower_state": (None, [vp, _dp]),
            "ref_quat_exp": (None, [_dp, _dp]),
        }
        u64 = C.c_uint64
        # robot/, empirical/, sim/session (ref_robot.cpp)
        sig.update({
            "ref_robot_last_error": (C.c_char_p, []),
            "ref_model_build": (vp, [C.c_char_p]),
            "ref_model_destroy": (None, [vp]),
            "ref_model_info": (None, [vp, _ip]),
            "ref_model_links": (None, [vp, _dp]),
            "ref_model_bladder": (None, [vp, _dp]),
            "ref_model_mesh": (None, [vp, _dp, _ip, _dp]),
            "ref_skeleton_validate": (C.c_int, [C.c_int, _dp]),
            "ref_samples_create": (vp, [vp, C.c_double, u64]),
            "ref_samples_destroy": (None, [vp]),
            "ref_samples_n": (C.c_int64, [vp]),
            "ref_samples_get": (None, [vp, _dp, _dp, _dp, _dp]),
            "ref_kinematics": (None, [vp, _dp, _dp]),
            "ref_mass_matrix": (None, [vp, _dp, _dp]),
            "ref_bias_forces": (None, [vp, _dp, _dp, _dp]),
            "ref_robot_step": (C.c_int, [vp, _dp, _dp, _dp, C.c_double, _dp, C.c_double,
                                         C.c_double, C.c_int]),
            "ref_update_samples": (None, [vp, vp, _dp, _dp, _dp, _dp]),
            "ref_skinned_tau": (None, [vp, vp, _dp, _dp, _ip, _dp, _dp]),
            "ref_emp_create": (vp, [C.c_double, C.c_int, C.c_double, _dp, C.c_double, C.c_double]),
            "ref_emp_destroy": (None, [vp]),
            "ref_emp_add_robot": (C.c_int, [vp, vp, _dp, C.c_double, u64]),
            "ref_be_set_actuation": (None, [vp, C.c_int, C.c_int, _dp]),
            "ref_be_change_bladder": (None, [vp, C.c_int, C.c_int, C.c_double]),
            "ref_be_step": (C.c_int, [vp, C.c_int, _ip]),
            "ref_be_robot": (None, [vp, C.c_int, C.c_int, _dp, _dp, _dp, _dp]),
            "ref_be_set_state": (None, [vp, C.c_int, C.c_int, _dp]),
            "ref_be_samples": (None, [vp, C.c_int, C.c_int, _dp, _dp, _dp]),
            "ref_be_n_samples": (C.c_int64, [vp, C.c_int, C.c_int]),
            "ref_cs_create": (vp, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                   C.c_double, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                   _dp, C.c_int, C.c_double, C.c_int]),
            "ref_cs_destroy": (None, [vp]),
            "ref_cs_add_robot": (C.c_int, [vp, vp, _dp, C.c_double, u64]),
            "ref_cs_frame": (None, [vp, _dp]),
            "ref_cs_get_f": (None, [vp, _dp]),
            "ref_cs_macro": (None, [vp, _dp, _dp]),
        })
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _ref = lib
    return _ref


# --------------------------------------------------------------------------
# Reference Rng (core/rng.hpp:14-84), restated in numpy for seeding inputs.
_M64 = (1 << 64) - 1


class Rng:
    """xoshiro256** with splitmix64 seeding (rng.hpp:14-84), bit-identical to the reference."""

    def __init__(self, seed: int = 0):
        self.s = [0, 0, 0, 0]
        x = seed & _M64
        for k in range(4):
            x = (x + 0x9E3779B97F4A7C15) & _M64
            z = x
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
            self.s[k] = z ^ (z >> 31)

    @staticmethod
    def _rotl(x, k):
        return ((x << k) | (x >> (64 - k))) & _M64

    def next_u64(self) -> int:
        s = self.s
        result = (self._rotl((s[1] * 5) & _M64, 7) * 9) & _M64
        t = (s[1] << 17) & _M64
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = self._rotl(s[3], 45)
        return result

    def uniform(self, lo: float | None = None, hi: float | None = None) -> float:
        u = (self.next_u64() >> 11) * (2.0 ** -53)
        if lo is None:
            return u
        return lo + (hi - lo) * u

    def uniforms(self, n: int) -> np.ndarray:
        return np.array([self.uniform() for _ in range(n)], dtype=np.float64)


# --------------------------------------------------------------------------
# Articulated dynamics restated (fsg_dyn_oracle.c; dynamics.hpp).  Robots and
# states are the product's host types (paper_2206_01683_b200.dynamics), whose
# POD structs are the boundary's own layout.
class DynKC(C.Structure):
    _L = 12
    _fields_ = [("E", (C.c_double * 9) * _L), ("r", (C.c_double * 3) * _L),
                ("R_world", (C.c_double * 9) * _L), ("p_world", (C.c_double * 3) * _L),
                ("v_body", (C.c_double * 6) * _L), ("omega_world", (C.c_double * 3) * _L),
                ("v_origin_world", (C.c_double * 3) * _L)]


class DynOracle:
    """One robot (host types from paper_2206_01683_b200.dynamics) on the fp64
    restatement; states are JointState objects, updated in place by step()."""

    def __init__(self, robot):
        self.robot = robot
        self.rs = robot.to_struct()
        self.nd, self.nj = robot.n_dofs, robot.n_joints
        self.bladder_volume = robot.bladder.volume

    def _st(self, st):
        return st.to_struct()

    def _back(self, s, st):
        from paper_2206_01683_b200.dynamics import JointState
        n = JointState.from_struct(s, self.nj, self.nd)
        st.base_pos, st.base_quat, st.q, st.v, st.qdd = n.base_pos, n.base_quat, n.q, n.v, n.qdd

    def kinematics(self, st):
        kc = DynKC()
        oracle().orc_forward_kinematics(C.byref(self.rs), C.byref(self._st(st)), C.byref(kc))
        return kc

    def mass_matrix(self, st):
        M = np.zeros(self.nd * self.nd)
        oracle().orc_mass_matrix(C.byref(self.rs), C.byref(self.kinematics(st)), dptr(M))
        return M.reshape(self.nd, self.nd)

    def bias_forces(self, st, g=(0.0, 0.0, 0.0)):
        c = np.zeros(max(self.nd, 1))
        s = self._st(st)
        kc = DynKC()
        oracle().orc_forward_kinematics(C.byref(self.rs), C.byref(s), C.byref(kc))
        oracle().orc_bias_forces(C.byref(self.rs), C.byref(s), C.byref(kc), dptr(d3(g)), dptr(c))
        return c[: self.nd]

    def internal_forces(self, st, act):
        tau = np.zeros(max(self.nd, 1))
        cl = oracle().orc_internal_forces(C.byref(self.rs), C.byref(self._st(st)),
                                          dptr(d3(act) if len(act) else np.zeros(1)), dptr(tau))
        return tau[: self.nd], bool(cl)

    def joint_limit_forces(self, st):
        tau = np.zeros(max(self.nd, 1))
        oracle().orc_joint_limit_forces(C.byref(self.rs), C.byref(self._st(st)), dptr(tau))
        return tau[: self.nd]

    def forward_dynamics(self, st, tau_int, tau_ext, g=(0.0, 0.0, 0.0)):
        qdd = np.zeros(self.nd)
        ok = oracle().orc_forward_dynamics(C.byref(self.rs), C.byref(self._st(st)), dptr(d3(tau_int)),
                                           dptr(d3(tau_ext)), dptr(d3(g)), dptr(qdd))
        if not ok:
            raise ArithmeticError("mass matrix is not positive definite; check link inertias")
        return qdd

    def buoyancy_gravity_forces(self, st, rho, g, bladder_volume=None):
        tau = np.zeros(max(self.nd, 1))
        bv = self.bladder_volume if bladder_volume is None else bladder_volume
        oracle().orc_buoyancy_gravity_forces(C.byref(self.rs), C.byref(self.kinematics(st)),
                                             float(bv), float(rho), dptr(d3(g)), dptr(tau))
        return tau[: self.nd]

    def integrate(self, st, act, tau_ext, dt, substeps=1, g=(0.0, 0.0, 0.0)):
        s = self._st(st)
        a = d3(act) if len(act) else np.zeros(1)
        fl = oracle().orc_integrate(C.byref(self.rs), C.byref(s), dptr(a), dptr(d3(tau_ext)),
                                    float(dt), int(substeps), dptr(d3(g)))
        self._back(s, st)
        return fl

    def robot_step(self, st, act, tau_ext, rho, g_hydro, dt, substeps=1, g=None):
        s = self._st(st)
        a = d3(act) if len(act) else np.zeros(1)
        fl = oracle().orc_robot_step(C.byref(self.rs), C.byref(s), float(self.bladder_volume), dptr(a),
                                     None if tau_ext is None else dptr(d3(tau_ext)), float(rho),
                                     None if g_hydro is None else dptr(d3(g_hydro)), float(dt),
                                     int(substeps), None if g is None else dptr(d3(g)))
        self._back(s, st)
        return fl

    def mechanical_energy(self, st, g):
        return oracle().orc_mechanical_energy(C.byref(self.rs), C.byref(self._st(st)), dptr(d3(g)))

    def pose(self, st, rest_R, rest_p):
        out = np.zeros(30 * 12)
        oracle().orc_dyn_pose(C.byref(self.rs), C.byref(self._st(st)), dptr(d3(rest_R)), dptr(d3(rest_p)),
                              out.ctypes.data_as(C.c_void_p))
        return out


def quat_exp(w):
    q = np.zeros(4)
    oracle().orc_quat_exp(dptr(d3(w)), dptr(q))
    return q


def quat_to_R(q):
    R = np.zeros(9)
    oracle().orc_quat_to_R(dptr(d3(q)), dptr(R))
    return R.reshape(3, 3)
