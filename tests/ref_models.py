"""The reference's own robot models, run through oracle/_ref -- TEST INFRASTRUCTURE.

``RefModel("koi" | "eel" | "flatfish")`` is build_fish_model(<design>())
(model_builder.hpp:104-264) compiled unmodified into oracle/_ref/libfishref.so
(oracle/ref_robot.cpp).  It exposes the reference's

* skeleton as the product's host type (``robot()`` -> dynamics.Robot), so the
  device dynamics and skinning run on exactly the reference's link masses,
  inertias, joint frames and bladder;
* ``samples(spacing, seed)``: robot::sample_surface (sampling.hpp:164-303);
* ``step``: the robot half of CoupledSession::step (session.hpp:167-175);
* ``update_samples`` / ``skinned_tau``: sampling.hpp:307-322 and the tau_ext
  loop of session.hpp:127-143;
* ``EmpiricalRef`` / ``SessionRef``: empirical::EmpiricalBackend and
  sim::CoupledSession themselves.

Packed joint state: base_pos[3], base_quat[4] (w,x,y,z), q[nj], v[nd].
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from oracle import bind as B

dptr, iptr = B.dptr, B.iptr


def _err():
    return B.ref().ref_robot_last_error().decode()


# -- conversions from the packed reference layouts (work without _ref: goldens) --
def robot_from_packed(links, bladder):
    """dynamics.Robot with the reference's links and bladder, value for value."""
    from paper_2206_01683_b200 import dynamics as D
    out = []
    for o in np.asarray(links, dtype=np.float64):
        out.append(D.Link(parent=int(o[0]), joint=int(o[1]), joint_origin=o[2:5].copy(),
                          joint_rotation=o[5:14].reshape(3, 3).copy(), axis=o[14:17].copy(),
                          mass=float(o[17]), com=o[18:21].copy(),
                          inertia_com=o[21:30].reshape(3, 3).copy(), stiffness=float(o[30]),
                          damping=float(o[31]), q_rest=float(o[32]), limit_lo=float(o[33]),
                          limit_hi=float(o[34]), torque_limit=float(o[35]),
                          displaced_volume=float(o[36]), volume_centroid=o[37:40].copy()))
    b = np.asarray(bladder, dtype=np.float64)
    return D.Robot(out, D.Bladder(volume=float(b[0]), volume_min=float(b[1]),
                                  volume_max=float(b[2]), rate_bound=float(b[3]),
                                  centroid=b[4:7].copy()))


def skeleton_from_packed(links):
    """session.Skeleton (the skinning topology, fsg_skeleton) of packed links."""
    from paper_2206_01683_b200.session import Skeleton
    r = robot_from_packed(links, np.zeros(8))
    parent = [l.parent for l in r.links]
    dofi = [r.dof_index(i) for i in range(r.n_links)]
    axis = np.array([np.asarray(l.axis) / np.linalg.norm(l.axis) for l in r.links])
    return Skeleton(parent, dofi, axis, r.floating_base, r.n_dofs)


def pose_from_kc(kc) -> np.ndarray:
    """fsg_body_pose (packed) from ref_kinematics rows [n_links, 30]."""
    from paper_2206_01683_b200._abi import SKIN_MAX_LINKS
    k = np.asarray(kc, dtype=np.float64)
    Lm, n = SKIN_MAX_LINKS, k.shape[0]
    out = np.zeros(30 * Lm)
    out[0:9 * n] = k[:, 18:27].reshape(-1)                       # bone_R
    out[9 * Lm:9 * Lm + 3 * n] = k[:, 27:30].reshape(-1)         # bone_t
    out[12 * Lm:12 * Lm + 9 * n] = k[:, 0:9].reshape(-1)         # R_world
    out[21 * Lm:21 * Lm + 3 * n] = k[:, 9:12].reshape(-1)        # p_world
    out[24 * Lm:24 * Lm + 3 * n] = k[:, 12:15].reshape(-1)       # v_origin_world
    out[27 * Lm:27 * Lm + 3 * n] = k[:, 15:18].reshape(-1)       # omega_world
    return out


def unpack_state(x, n_joints, n_dofs):
    from paper_2206_01683_b200.dynamics import JointState
    x = np.asarray(x, dtype=np.float64)
    return JointState(x[0:3].copy(), x[3:7].copy(), x[7:7 + n_joints].copy(),
                      x[7 + n_joints:7 + n_joints + n_dofs].copy(), np.zeros(n_dofs))


def pack_state(st) -> np.ndarray:
    return np.concatenate([st.base_pos, st.base_quat, st.q, st.v]).astype(np.float64)


class RefModel:
    def __init__(self, design: str):
        self.L = B.ref()
        self.design = design
        self.h = self.L.ref_model_build(design.encode())
        if not self.h:
            raise RuntimeError(_err())
        info = np.zeros(6, dtype=np.int32)
        self.L.ref_model_info(self.h, iptr(info))
        self.n_links, self.n_joints, self.n_dofs, self.floating, self.nv, self.nt = map(int, info)
        self.links = np.zeros((self.n_links, 40))
        self.L.ref_model_links(self.h, dptr(self.links))
        self.bladder = np.zeros(8)
        self.L.ref_model_bladder(self.h, dptr(self.bladder))

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_model_destroy(self.h)
            self.h = None

    def robot(self):
        """dynamics.Robot with the reference's links and bladder, value for value."""
        return robot_from_packed(self.links, self.bladder)

    def skeleton(self):
        """session.Skeleton (the skinning topology, fsg_skeleton) of this model."""
        return skeleton_from_packed(self.links)

    def samples(self, spacing: float, seed: int = 1234):
        """-> (rest_points [m,3], rest_normals [m,3], areas [m], weights [m, n_links])."""
        h = self.L.ref_samples_create(self.h, float(spacing), int(seed))
        if not h:
            raise RuntimeError(_err())
        m = int(self.L.ref_samples_n(h))
        P, N, A, W = np.zeros((m, 3)), np.zeros((m, 3)), np.zeros(m), np.zeros((m, self.n_links))
        self.L.ref_samples_get(h, dptr(P), dptr(N), dptr(A), dptr(W))
        self.L.ref_samples_destroy(h)
        return P, N, A, W

    # -- packed joint state ----------------------------------------------------
    def pack(self, st) -> np.ndarray:
        return np.concatenate([st.base_pos, st.base_quat, st.q, st.v]).astype(np.float64)

    def unpack(self, x):
        return unpack_state(x, self.n_joints, self.n_dofs)

    def zero_state(self) -> np.ndarray:
        x = np.zeros(7 + self.n_joints + self.n_dofs)
        x[3] = 1.0
        return x

    # -- the reference's functions --------------------------------------------
    def step(self, x, actuation, tau_ext=None, rho=1000.0, g_hydro=(0.0, 0.0, -9.81),
             bladder_volume=-1.0, dt=0.004, substeps=4) -> int:
        """In place on the packed state x; returns 1 on NumericalError."""
        return self.L.ref_robot_step(self.h, dptr(x), dptr(B.d3(actuation) if len(actuation) else
                                                          np.zeros(1)),
                                     None if tau_ext is None else dptr(B.d3(tau_ext)), float(rho),
                                     dptr(B.d3(g_hydro)), float(bladder_volume), float(dt),
                                     int(substeps))

    def kinematics(self, x):
        """per link (R_world [3,3], p_world, v_origin_world, omega_world, bone_R, bone_t)"""
        out = np.zeros((self.n_links, 30))
        self.L.ref_kinematics(self.h, dptr(B.d3(x)), dptr(out))
        return out

    def pose(self, x) -> np.ndarray:
        """fsg_body_pose (packed) at state x."""
        return pose_from_kc(self.kinematics(x))

    def mass_matrix(self, x):
        M = np.zeros(self.n_dofs * self.n_dofs)
        self.L.ref_mass_matrix(self.h, dptr(B.d3(x)), dptr(M))
        return M.reshape(self.n_dofs, self.n_dofs).T  # column-major

    def bias_forces(self, x, g=(0.0, 0.0, 0.0)):
        c = np.zeros(self.n_dofs)
        self.L.ref_bias_forces(self.h, dptr(B.d3(x)), dptr(B.d3(g)), dptr(c))
        return c


class RefSamples:
    """One robot's SurfaceSamples inside the reference (for update_samples /
    skinned_tau at arbitrary states)."""

    def __init__(self, model: RefModel, spacing: float, seed: int = 1234):
        self.model, self.L = model, model.L
        self.h = self.L.ref_samples_create(model.h, float(spacing), int(seed))
        if not self.h:
            raise RuntimeError(_err())
        self.m = int(self.L.ref_samples_n(self.h))

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_samples_destroy(self.h)
            self.h = None

    def update(self, x):
        P, V, N = (np.zeros((self.m, 3)) for _ in range(3))
        self.L.ref_update_samples(self.model.h, self.h, dptr(B.d3(x)), dptr(P), dptr(V), dptr(N))
        return P, V, N

    def skinned_tau(self, x, f_world, valid):
        tau, stats = np.zeros(self.model.n_dofs), np.zeros(8)
        self.L.ref_skinned_tau(self.model.h, self.h, dptr(B.d3(x)),
                               dptr(np.ascontiguousarray(f_world, dtype=np.float64).reshape(-1)),
                               iptr(np.ascontiguousarray(valid, dtype=np.int32)), dptr(tau),
                               dptr(stats))
        return tau, stats


class _Backend:
    kind = -1

    def set_actuation(self, i, act):
        a = B.d3(act) if len(act) else np.zeros(1)
        self.L.ref_be_set_actuation(self.h, self.kind, int(i), dptr(a))

    def change_bladder(self, i, dv):
        self.L.ref_be_change_bladder(self.h, self.kind, int(i), float(dv))

    def step(self):
        oob = C.c_int(0)
        r = self.L.ref_be_step(self.h, self.kind, C.byref(oob))
        if r < 0:
            raise RuntimeError(_err())
        return bool(r), int(oob.value)

    def robot(self, i):
        m = self.models[i]
        x = np.zeros(7 + m.n_joints + m.n_dofs)
        tau, stats, bv = np.zeros(m.n_dofs), np.zeros(8), C.c_double(0)
        self.L.ref_be_robot(self.h, self.kind, int(i), dptr(x), dptr(tau), dptr(stats),
                            C.byref(bv))
        return x, tau, stats, float(bv.value)

    def set_state(self, i, x):
        self.L.ref_be_set_state(self.h, self.kind, int(i), dptr(B.d3(x)))

    def samples(self, i):
        n = int(self.L.ref_be_n_samples(self.h, self.kind, int(i)))
        P, V, N = (np.zeros((n, 3)) for _ in range(3))
        self.L.ref_be_samples(self.h, self.kind, int(i), dptr(P), dptr(V), dptr(N))
        return P, V, N

    def add_robot(self, model: RefModel, pos=(0.0, 0.0, 0.0), yaw=0.0, seed=1234):
        r = self._add(self.h, model.h, dptr(B.d3(pos)), float(yaw), int(seed))
        if r < 0:
            raise RuntimeError(_err())
        self.models.append(model)
        return r


class EmpiricalRef(_Backend):
    """empirical::EmpiricalBackend (empirical.hpp:36-110), the reference's own."""

    kind = 0

    def __init__(self, dt=0.004, substeps=4, rho=1000.0, gravity=(0.0, 0.0, -9.81),
                 spacing=0.02, k=40.0):
        self.L = B.ref()
        self.models = []
        self.h = self.L.ref_emp_create(float(dt), int(substeps), float(rho),
                                       dptr(B.d3(gravity)), float(spacing), float(k))
        if not self.h:
            raise RuntimeError(_err())
        self._add = self.L.ref_emp_add_robot

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_emp_destroy(self.h)
            self.h = None


class SessionRef(_Backend):
    """sim::CoupledSession (session.hpp:29-241), the reference's own."""

    kind = 1

    def __init__(self, dims, dx, dt, rho=1000.0, nu=1e-6, kernel=0, wall=0, frame_mode=2,
                 frame_tc=0.2, recenter_cells=2.0, gravity=(0.0, 0.0, -9.81), substeps=4,
                 marker_spacing=0.0, tracked=0):
        self.L = B.ref()
        self.models = []
        self.dims = tuple(int(d) for d in dims)
        self.h = self.L.ref_cs_create(*self.dims, float(dx), float(dt), float(rho), float(nu),
                                      int(kernel), int(wall), int(frame_mode), float(frame_tc),
                                      float(recenter_cells), dptr(B.d3(gravity)), int(substeps),
                                      float(marker_spacing), int(tracked))
        if not self.h:
            raise RuntimeError(_err())
        self._add = self.L.ref_cs_add_robot

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_cs_destroy(self.h)
            self.h = None

    def frame(self):
        out = np.zeros(19)
        self.L.ref_cs_frame(self.h, dptr(out))
        return out

    def get_f(self):
        n = int(np.prod(self.dims))
        f = np.zeros(19 * n)
        self.L.ref_cs_get_f(self.h, dptr(f))
        return f

    def macro(self):
        n = int(np.prod(self.dims))
        rho, u = np.zeros(n), np.zeros(3 * n)
        self.L.ref_cs_macro(self.h, dptr(rho), dptr(u))
        return rho, u.reshape(n, 3)
