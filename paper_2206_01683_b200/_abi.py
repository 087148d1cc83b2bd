"""ctypes binding of the C ABI in include/fsg.h (libfsg.so, built in-tree).

There is deliberately no fallback: if libfsg.so is missing or no CUDA device
is visible the calls fail loudly (FsgError).  The CPU oracle lives in
oracle/ and is never imported from here.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PEER_HANDLE_BYTES = 512  # FSG_PEER_HANDLE_BYTES (include/fsg.h)

# FSG_LIB: alternative build of the same ABI (dev A/B runs); the default is the in-tree libfsg.so
LIB_PATH = os.environ.get("FSG_LIB") or os.path.join(HERE, "libfsg.so")

FSG_OK, FSG_EINPUT, FSG_ECUDA, FSG_ESTATE = 0, 1, 2, 3


class FsgError(RuntimeError):
    """Raised for every non-zero fsg_* return code."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[fsg code {code}] {msg}")
        self.code = code


class InputError(FsgError, ValueError):
    """Invalid configuration (the reference throws fishsim::InputError, types.hpp:27-30)."""


class fsg_config(C.Structure):
    _fields_ = [("dims", C.c_int * 3), ("dx", C.c_double), ("dt", C.c_double),
                ("rho", C.c_double), ("nu", C.c_double), ("boundary", C.c_int),
                ("kernel", C.c_int), ("wall", C.c_int), ("frame_mode", C.c_int),
                ("precision", C.c_int), ("device", C.c_int), ("max_markers", C.c_int),
                ("z_offset", C.c_int), ("nz_global", C.c_int)]


class fsg_status(C.Structure):
    _fields_ = [("finite", C.c_int), ("min_f", C.c_double), ("n_nonpositive_rho", C.c_int),
                ("out_of_bounds_markers", C.c_int), ("stable", C.c_int)]


class fsg_frame_state(C.Structure):
    _fields_ = [("p", C.c_double * 3), ("pd", C.c_double * 3), ("pdd", C.c_double * 3),
                ("q", C.c_double * 4), ("omega", C.c_double * 3), ("alpha", C.c_double * 3)]


SKIN_MAX_LINKS, SKIN_MAX_BODIES, SKIN_MAX_WEIGHTS = 12, 4, 4
_L = SKIN_MAX_LINKS


class fsg_skeleton(C.Structure):
    _fields_ = [("n_links", C.c_int), ("floating_base", C.c_int), ("n_dofs", C.c_int),
                ("parent", C.c_int * _L), ("dof_index", C.c_int * _L),
                ("axis", (C.c_double * 3) * _L)]


class fsg_body_pose(C.Structure):
    _fields_ = [("bone_R", (C.c_double * 9) * _L), ("bone_t", (C.c_double * 3) * _L),
                ("R_world", (C.c_double * 9) * _L), ("p_world", (C.c_double * 3) * _L),
                ("v_origin_world", (C.c_double * 3) * _L), ("omega_world", (C.c_double * 3) * _L)]


DYN_MAX_LINKS = 12
DYN_MAX_DOFS = 6 + DYN_MAX_LINKS
FSG_JOINT_FREE, FSG_JOINT_REVOLUTE, FSG_JOINT_FIXED = 0, 1, 2
FSG_DYN_CLAMPED, FSG_DYN_NOT_SPD, FSG_DYN_NONFINITE = 1, 2, 4


class fsg_link(C.Structure):
    _fields_ = [("parent", C.c_int), ("joint", C.c_int), ("joint_origin", C.c_double * 3),
                ("joint_rotation", C.c_double * 9), ("axis", C.c_double * 3), ("mass", C.c_double),
                ("com", C.c_double * 3), ("inertia_com", C.c_double * 9), ("stiffness", C.c_double),
                ("damping", C.c_double), ("q_rest", C.c_double), ("limit_lo", C.c_double),
                ("limit_hi", C.c_double), ("torque_limit", C.c_double),
                ("displaced_volume", C.c_double), ("volume_centroid", C.c_double * 3)]


class fsg_robot(C.Structure):
    _fields_ = [("n_links", C.c_int), ("links", fsg_link * DYN_MAX_LINKS),
                ("bladder_volume", C.c_double), ("bladder_volume_min", C.c_double),
                ("bladder_volume_max", C.c_double), ("bladder_rate_bound", C.c_double),
                ("bladder_centroid", C.c_double * 3)]


class fsg_joint_state(C.Structure):
    _fields_ = [("base_pos", C.c_double * 3), ("base_quat", C.c_double * 4),
                ("q", C.c_double * DYN_MAX_LINKS), ("v", C.c_double * DYN_MAX_DOFS),
                ("qdd", C.c_double * DYN_MAX_DOFS)]


_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_i64p = C.POINTER(C.c_int64)
_vp = C.c_void_p

# name -> (restype, argtypes); this is the complete exported surface of fsg.h
SIGNATURES = {
    "fsg_last_error": (C.c_char_p, []),
    "fsg_abi_version": (C.c_int, []),
    "fsg_config_default": (None, [C.POINTER(fsg_config)]),
    "fsg_tau": (C.c_double, [C.c_double, C.c_double, C.c_double]),
    "fsg_create": (C.c_int, [C.POINTER(fsg_config), C.POINTER(_vp)]),
    "fsg_destroy": (C.c_int, [_vp]),
    "fsg_stream": (_vp, [_vp]),
    "fsg_reset_rest": (C.c_int, [_vp]),
    "fsg_initialize": (C.c_int, [_vp, _dp, _dp]),
    "fsg_set_f": (C.c_int, [_vp, _dp]),
    "fsg_get_f": (C.c_int, [_vp, _dp]),
    "fsg_set_force": (C.c_int, [_vp, _dp]),
    "fsg_collide_and_stream": (C.c_int, [_vp, C.POINTER(fsg_status)]),
    "fsg_macroscopic": (C.c_int, [_vp, _dp, _dp, _ip]),
    "fsg_total_mass": (C.c_int, [_vp, _dp]),
    "fsg_total_momentum": (C.c_int, [_vp, _dp]),
    "fsg_set_frame": (C.c_int, [_vp, C.POINTER(fsg_frame_state)]),
    "fsg_get_frame": (C.c_int, [_vp, C.POINTER(fsg_frame_state)]),
    "fsg_recenter": (C.c_int, [_vp, _ip]),
    "fsg_set_markers": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, _vp, _vp]),
    "fsg_set_markers_device": (C.c_int, [_vp, C.c_int, _i64p, _vp, _vp, _vp, _vp]),
    "fsg_step": (C.c_int, [_vp, C.POINTER(fsg_status)]),
    "fsg_step_async": (C.c_int, [_vp]),
    "fsg_last_status": (C.c_int, [_vp, C.POINTER(fsg_status)]),
    "fsg_get_marker_forces": (C.c_int, [_vp, _vp, _vp, _vp]),
    "fsg_get_macro": (C.c_int, [_vp, _dp, _dp]),
    "fsg_get_force": (C.c_int, [_vp, _dp]),
    "fsg_set_force_capture": (C.c_int, [_vp, C.c_int]),
    "fsg_get_stencils": (C.c_int, [_vp, _ip]),
    "fsg_set_skin": (C.c_int, [_vp, C.c_int, _i64p, C.POINTER(fsg_skeleton), _dp, _dp, _dp, _dp]),
    "fsg_set_pose": (C.c_int, [_vp, C.POINTER(fsg_body_pose)]),
    "fsg_get_body_wrench": (C.c_int, [_vp, _vp, _vp]),
    "fsg_get_markers": (C.c_int, [_vp, _dp, _dp, _dp]),
    "fsg_step_skinned": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "fsg_drag_last_error": (C.c_char_p, []),
    "fsg_drag_create": (C.c_int, [C.c_int, C.c_double, C.c_int, C.c_int, C.POINTER(_vp)]),
    "fsg_drag_destroy": (C.c_int, [_vp]),
    "fsg_drag_set_skin": (C.c_int, [_vp, C.c_int, C.POINTER(fsg_skeleton), C.c_int, _dp, _dp, _dp, _dp]),
    "fsg_drag_set_pose": (C.c_int, [_vp, C.c_int, _vp]),
    "fsg_drag_set_poses": (C.c_int, [_vp, _vp]),
    "fsg_drag_step": (C.c_int, [_vp, _dp, _dp]),
    "fsg_dyn_last_error": (C.c_char_p, []),
    "fsg_dyn_create": (C.c_int, [C.POINTER(fsg_robot), C.c_int, C.c_int, C.POINTER(_vp)]),
    "fsg_dyn_destroy": (C.c_int, [_vp]),
    "fsg_dyn_n_dofs": (C.c_int, [_vp]),
    "fsg_dyn_n_joints": (C.c_int, [_vp]),
    "fsg_dyn_set_state": (C.c_int, [_vp, _vp]),
    "fsg_dyn_get_state": (C.c_int, [_vp, _vp]),
    "fsg_dyn_change_bladder": (C.c_int, [_vp, _dp, _dp]),
    "fsg_dyn_step": (C.c_int, [_vp, _dp, _dp, C.c_double, _dp, C.c_double, C.c_int, _dp, _ip]),
    "fsg_dyn_step_device": (C.c_int, [_vp, _vp, _vp, C.c_double, _dp, C.c_double, C.c_int, _dp,
                                      _vp]),
    "fsg_dyn_mass_matrix": (C.c_int, [_vp, _dp, _dp, _dp]),
    "fsg_dyn_poses": (C.c_int, [_vp, _dp, _dp, _vp]),
    "fsg_dyn_set_rest": (C.c_int, [_vp, _dp, _dp]),
    "fsg_snapshot_begin": (C.c_int, [_vp]),
    "fsg_snapshot_wait": (C.c_int, [_vp, _dp, _dp]),
    "fsg_write_vtk": (C.c_int, [_vp, C.c_char_p, _dp]),
    "fsg_io_last_error": (C.c_char_p, []),
    "fsg_write_vtk_fields": (C.c_int, [C.c_char_p, _ip, _dp, _dp, C.c_double, C.c_double, C.c_double,
                                       _dp]),
    "fsg_format_full": (C.c_int, [C.c_double, C.c_char_p, C.c_int]),
    "fsg_csv_open": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_char_p), C.POINTER(_vp)]),
    "fsg_csv_write_row": (C.c_int, [_vp, C.c_int, _dp]),
    "fsg_csv_close": (C.c_int, [_vp]),
    "fsg_profile_enable": (C.c_int, [_vp, C.c_int]),
    "fsg_profile_read": (C.c_int, [_vp, _dp, _ip]),
    "fsg_follower_create": (C.c_int, [C.c_int, C.c_double, C.POINTER(_vp)]),
    "fsg_follower_destroy": (C.c_int, [_vp]),
    "fsg_follower_reset": (C.c_int, [_vp, _dp, C.c_double]),
    "fsg_follower_step": (C.c_int, [_vp, _dp, _dp, C.c_double]),
    "fsg_follower_state": (C.c_int, [_vp, C.POINTER(fsg_frame_state)]),
    "fsg_follower_set_state": (C.c_int, [_vp, C.POINTER(fsg_frame_state)]),
    "fsg_follower_center": (C.c_int, [_vp, _dp, _dp]),
    "fsg_batch_set_follow": (C.c_int, [_vp, C.c_double, C.c_double]),
    "fsg_batch_center_frames": (C.c_int, [_vp, _vp]),
    "fsg_batch_last_shifts": (C.c_int, [_vp, _vp]),
    "fsg_batch_create": (C.c_int, [C.POINTER(fsg_config), C.c_int, C.POINTER(_vp)]),
    "fsg_batch_destroy": (C.c_int, [_vp]),
    "fsg_batch_session": (_vp, [_vp, C.c_int]),
    "fsg_batch_step_async": (C.c_int, [_vp]),
    "fsg_batch_step": (C.c_int, [_vp, C.POINTER(fsg_status)]),
    "fsg_batch_step_skinned": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "fsg_batch_step_dynamic": (C.c_int, [_vp, _vp, _vp, _dp, C.c_double, _dp, C.c_double, C.c_int,
                                         _vp, _vp, _vp]),
    "fsg_halo_bytes": (C.c_size_t, [_vp]),
    "fsg_halo_pack": (C.c_int, [_vp, _vp, _vp]),
    "fsg_halo_unpack": (C.c_int, [_vp, _vp, _vp]),
    "fsg_halo_buffers": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp),
                                   C.POINTER(_vp)]),
    "fsg_halo_begin": (C.c_int, [_vp, _vp]),
    "fsg_halo_end": (C.c_int, [_vp, _vp, C.c_int, C.c_int]),
    "fsg_peer_export": (C.c_int, [_vp, C.c_char_p]),
    "fsg_peer_connect": (C.c_int, [_vp, C.c_char_p, C.c_char_p]),
    "fsg_peer_disconnect": (C.c_int, [_vp]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libfsg.so (raises if it was not built: there is no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FsgError(FSG_ECUDA, f"{LIB_PATH} not built; run __graft_entry__.build() "
                                      "(the B200 path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int, drag: bool = False, io: bool = False, dyn: bool = False) -> None:
    if rc != FSG_OK:
        L = lib()
        err = L.fsg_drag_last_error if drag else (L.fsg_io_last_error if io else L.fsg_last_error)
        if dyn:
            err = L.fsg_dyn_last_error
        msg = err().decode(errors="replace")
        if rc == FSG_EINPUT:
            raise InputError(rc, msg)
        raise FsgError(rc, msg)


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    if a.dtype != np.float64 or not a.flags.c_contiguous:
        raise TypeError("expected a C-contiguous float64 array")
    return a.ctypes.data_as(_dp)


def iptr(a: np.ndarray | None):
    if a is None:
        return None
    if a.dtype != np.int32 or not a.flags.c_contiguous:
        raise TypeError("expected a C-contiguous int32 array")
    return a.ctypes.data_as(_ip)
