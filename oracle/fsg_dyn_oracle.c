/* fsg_dyn_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * fp64 restatement of the reference's articulated-body dynamics
 * (fishsim/robot/dynamics.hpp, spatial.hpp, skeleton.hpp; quat_exp in
 * core/types.hpp), used to check the device robot step (fsg_dyn_*).  The
 * reference's robot/ headers need dynamic Eigen (VectorXd/MatrixXd blocks,
 * LLT, SelfAdjointEigenSolver), which the oracle's Eigen stand-in does not
 * supply, so this restatement is pinned instead by the reference's own robot
 * tests (test_robot.cpp:69-343), restated in tests/test_dyn_oracle.py.
 * Vector algebra in plain coefficient order; Mat3/Mat6 row-major.  Compile
 * with -ffp-contract=off (oracle/Makefile).
 */
#include "fsg_dyn_oracle.h"

#include <math.h>
#include <string.h>

#define L FSG_DYN_MAX_LINKS
#define ND FSG_DYN_MAX_DOFS

/* ---- small algebra ------------------------------------------------------ */
static void mv3(const double* A, const double* x, double* y) {
  for (int i = 0; i < 3; ++i) y[i] = A[3 * i] * x[0] + A[3 * i + 1] * x[1] + A[3 * i + 2] * x[2];
}
static void mtv3(const double* A, const double* x, double* y) { /* A^T x */
  for (int i = 0; i < 3; ++i) y[i] = A[i] * x[0] + A[3 + i] * x[1] + A[6 + i] * x[2];
}
static void mm3(const double* A, const double* B, double* C) {
  double t[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      t[3 * i + j] = A[3 * i] * B[j] + A[3 * i + 1] * B[3 + j] + A[3 * i + 2] * B[6 + j];
  memcpy(C, t, sizeof t);
}
static void tr3(const double* A, double* T) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) T[3 * j + i] = A[3 * i + j];
}
static void cross3(const double* a, const double* b, double* c) {
  const double c0 = a[1] * b[2] - a[2] * b[1];
  const double c1 = a[2] * b[0] - a[0] * b[2];
  const double c2 = a[0] * b[1] - a[1] * b[0];
  c[0] = c0;
  c[1] = c1;
  c[2] = c2;
}
static double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static double dot6(const double* a, const double* b) {
  double s = 0.0;
  for (int k = 0; k < 6; ++k) s += a[k] * b[k];
  return s;
}
static void mv6(const double* A, const double* x, double* y) {
  for (int i = 0; i < 6; ++i) {
    double s = 0.0;
    for (int k = 0; k < 6; ++k) s += A[6 * i + k] * x[k];
    y[i] = s;
  }
}
static void normalized3(const double* a, double* o) {
  const double n = sqrt(dot3(a, a));
  o[0] = a[0] / n;
  o[1] = a[1] / n;
  o[2] = a[2] / n;
}
/* skew(v) (types.hpp:39-43) */
static void skew3(const double* v, double* m) {
  m[0] = 0.0, m[1] = -v[2], m[2] = v[1];
  m[3] = v[2], m[4] = 0.0, m[5] = -v[0];
  m[6] = -v[1], m[7] = v[0], m[8] = 0.0;
}

/* Quaternion::toRotationMatrix (Eigen 3.4 coefficient formulas), q = (w,x,y,z) */
void orc_quat_to_R(const double* q, double* R) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  const double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
  const double twx = tx * w, twy = ty * w, twz = tz * w;
  const double txx = tx * x, txy = ty * x, txz = tz * x;
  const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
  R[0] = 1.0 - (tyy + tzz), R[1] = txy - twz, R[2] = txz + twy;
  R[3] = txy + twz, R[4] = 1.0 - (txx + tzz), R[5] = tyz - twx;
  R[6] = txz - twy, R[7] = tyz + twx, R[8] = 1.0 - (txx + tyy);
}
/* AngleAxis::toRotationMatrix (Eigen 3.4), unit axis */
void orc_angle_axis_R(double angle, const double* a, double* R) {
  const double s = sin(angle), c = cos(angle);
  const double sa[3] = {s * a[0], s * a[1], s * a[2]};
  const double ca[3] = {(1.0 - c) * a[0], (1.0 - c) * a[1], (1.0 - c) * a[2]};
  double t;
  t = ca[0] * a[1];
  R[1] = t - sa[2];
  R[3] = t + sa[2];
  t = ca[0] * a[2];
  R[2] = t + sa[1];
  R[6] = t - sa[1];
  t = ca[1] * a[2];
  R[5] = t - sa[0];
  R[7] = t + sa[0];
  R[0] = ca[0] * a[0] + c;
  R[4] = ca[1] * a[1] + c;
  R[8] = ca[2] * a[2] + c;
}
static void quat_normalize(double* q) { /* stand-in pairing (x,z)+(y,w) */
  const double n = sqrt((q[1] * q[1] + q[3] * q[3]) + (q[2] * q[2] + q[0] * q[0]));
  for (int k = 0; k < 4; ++k) q[k] = q[k] / n;
}
static void quat_mul(const double* a, const double* b, double* o) {
  const double w = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
  const double x = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
  const double y = a[0] * b[2] + a[2] * b[0] + a[3] * b[1] - a[1] * b[3];
  const double z = a[0] * b[3] + a[3] * b[0] + a[1] * b[2] - a[2] * b[1];
  o[0] = w, o[1] = x, o[2] = y, o[3] = z;
}
/* quat_exp (types.hpp:71-79) */
void orc_quat_exp(const double* w, double* q) {
  const double angle = sqrt(dot3(w, w));
  if (angle < 1e-12) {
    q[0] = 1.0, q[1] = 0.5 * w[0], q[2] = 0.5 * w[1], q[3] = 0.5 * w[2];
    quat_normalize(q);
    return;
  }
  const double ax[3] = {w[0] / angle, w[1] / angle, w[2] / angle};
  const double ha = 0.5 * angle, s = sin(ha);
  q[0] = cos(ha), q[1] = s * ax[0], q[2] = s * ax[1], q[3] = s * ax[2];
}

/* ---- skeleton indexing (skeleton.hpp:60-93) ------------------------------ */
int orc_dyn_floating(const fsg_robot* r) { return r->n_links > 0 && r->links[0].joint == FSG_JOINT_FREE; }
int orc_dyn_n_joints(const fsg_robot* r) {
  int n = 0;
  for (int i = 1; i < r->n_links; ++i) n += r->links[i].joint == FSG_JOINT_REVOLUTE;
  return n;
}
int orc_dyn_n_dofs(const fsg_robot* r) { return (orc_dyn_floating(r) ? 6 : 0) + orc_dyn_n_joints(r); }
int orc_dyn_dof_index(const fsg_robot* r, int i) {
  if (i == 0) return orc_dyn_floating(r) ? 0 : -1;
  if (r->links[i].joint != FSG_JOINT_REVOLUTE) return -1;
  int idx = orc_dyn_floating(r) ? 6 : 0;
  for (int k = 1; k < i; ++k) idx += r->links[k].joint == FSG_JOINT_REVOLUTE;
  return idx;
}
static int joint_index(const fsg_robot* r, int i) {
  const int d = orc_dyn_dof_index(r, i);
  return d < 0 ? -1 : d - (orc_dyn_floating(r) ? 6 : 0);
}

/* ---- spatial algebra (spatial.hpp:15-80) ---------------------------------- */
static void apply_motion(const double* E, const double* r, const double* m, double* out) {
  double t[3], u[3], o[6];
  mv3(E, m, o);
  cross3(r, m, t);
  for (int k = 0; k < 3; ++k) u[k] = m[3 + k] - t[k];
  mv3(E, u, o + 3);
  memcpy(out, o, sizeof o);
}
static void transpose_force(const double* E, const double* r, const double* f, double* out) {
  double o[6], t[3];
  mtv3(E, f + 3, o + 3);
  mtv3(E, f, o);
  cross3(r, o + 3, t);
  for (int k = 0; k < 3; ++k) o[k] = o[k] + t[k];
  memcpy(out, o, sizeof o);
}
static void motion_matrix(const double* E, const double* r, double* X) {
  double S[9], ES[9];
  memset(X, 0, 36 * sizeof(double));
  skew3(r, S);
  mm3(E, S, ES);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      X[6 * i + j] = E[3 * i + j];
      X[6 * (i + 3) + j + 3] = E[3 * i + j];
      X[6 * (i + 3) + j] = -ES[3 * i + j];
    }
}
static void cross_motion(const double* v, const double* m, double* out) {
  double a[3], b[3], c[3];
  cross3(v, m, a);
  cross3(v, m + 3, b);
  cross3(v + 3, m, c);
  out[0] = a[0], out[1] = a[1], out[2] = a[2];
  for (int k = 0; k < 3; ++k) out[3 + k] = b[k] + c[k];
}
static void cross_force(const double* v, const double* f, double* out) {
  double a[3], b[3], c[3];
  cross3(v, f, a);
  cross3(v + 3, f + 3, b);
  cross3(v, f + 3, c);
  for (int k = 0; k < 3; ++k) out[k] = a[k] + b[k];
  out[3] = c[0], out[4] = c[1], out[5] = c[2];
}
void orc_spatial_inertia(double mass, const double* com, const double* Ic, double* I) {
  double c[9], ct[9], mc[9], mcct[9];
  skew3(com, c);
  tr3(c, ct);
  for (int k = 0; k < 9; ++k) mc[k] = mass * c[k];
  mm3(mc, ct, mcct);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      I[6 * i + j] = Ic[3 * i + j] + mcct[3 * i + j];
      I[6 * i + j + 3] = mc[3 * i + j];
      I[6 * (i + 3) + j] = mass * ct[3 * i + j];
      I[6 * (i + 3) + j + 3] = i == j ? mass : 0.0;
    }
}

/* ---- forward_kinematics (dynamics.hpp:23-63) ----------------------------- */
void orc_forward_kinematics(const fsg_robot* r, const fsg_joint_state* st, orc_kcache* kc) {
  const int nb = r->n_links;
  for (int i = 0; i < nb; ++i) {
    const fsg_link* l = &r->links[i];
    if (i == 0) {
      orc_quat_to_R(st->base_quat, kc->R_world[0]);
      memcpy(kc->p_world[0], st->base_pos, 3 * sizeof(double));
      tr3(kc->R_world[0], kc->E[0]);
      memcpy(kc->r[0], st->base_pos, 3 * sizeof(double));
      for (int k = 0; k < 6; ++k) kc->v_body[0][k] = orc_dyn_floating(r) ? st->v[k] : 0.0;
    } else {
      double rj[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, rrel[9], axis[3] = {0, 0, 0}, qd = 0.0, t[3];
      const int rev = l->joint == FSG_JOINT_REVOLUTE;
      if (rev) {
        normalized3(l->axis, axis);
        orc_angle_axis_R(st->q[joint_index(r, i)], axis, rj);
        qd = st->v[orc_dyn_dof_index(r, i)];
      }
      mm3(l->joint_rotation, rj, rrel);
      tr3(rrel, kc->E[i]);
      memcpy(kc->r[i], l->joint_origin, 3 * sizeof(double));
      const int pa = l->parent;
      mm3(kc->R_world[pa], rrel, kc->R_world[i]);
      mv3(kc->R_world[pa], l->joint_origin, t);
      for (int k = 0; k < 3; ++k) kc->p_world[i][k] = kc->p_world[pa][k] + t[k];
      apply_motion(kc->E[i], kc->r[i], kc->v_body[pa], kc->v_body[i]);
      if (rev)
        for (int k = 0; k < 3; ++k) kc->v_body[i][k] = kc->v_body[i][k] + axis[k] * qd;
    }
    mv3(kc->R_world[i], kc->v_body[i], kc->omega_world[i]);
    mv3(kc->R_world[i], kc->v_body[i] + 3, kc->v_origin_world[i]);
  }
}

/* ---- mass_matrix (CRBA, dynamics.hpp:72-114) ------------------------------ */
void orc_mass_matrix(const fsg_robot* r, const orc_kcache* kc, double* H) {
  const int nb = r->n_links, nd = orc_dyn_n_dofs(r);
  double ic[L][36];
  for (int i = 0; i < nb; ++i)
    orc_spatial_inertia(r->links[i].mass, r->links[i].com, r->links[i].inertia_com, ic[i]);
  for (int i = nb - 1; i >= 1; --i) {
    double X[36], T[36];
    motion_matrix(kc->E[i], kc->r[i], X);
    /* T = X^T ic[i]; ic[parent] += T X */
    for (int a = 0; a < 6; ++a)
      for (int b = 0; b < 6; ++b) {
        double s = 0.0;
        for (int k = 0; k < 6; ++k) s += X[6 * k + a] * ic[i][6 * k + b];
        T[6 * a + b] = s;
      }
    double* P = ic[r->links[i].parent];
    for (int a = 0; a < 6; ++a)
      for (int b = 0; b < 6; ++b) {
        double s = 0.0;
        for (int k = 0; k < 6; ++k) s += T[6 * a + k] * X[6 * k + b];
        P[6 * a + b] = P[6 * a + b] + s;
      }
  }
  memset(H, 0, (size_t)nd * nd * sizeof(double));
  if (orc_dyn_floating(r))
    for (int a = 0; a < 6; ++a)
      for (int b = 0; b < 6; ++b) H[nd * a + b] = ic[0][6 * a + b];
  for (int i = 1; i < nb; ++i) {
    if (r->links[i].joint != FSG_JOINT_REVOLUTE) continue;
    const int di = orc_dyn_dof_index(r, i);
    double s[6] = {0, 0, 0, 0, 0, 0}, f[6];
    normalized3(r->links[i].axis, s);
    mv6(ic[i], s, f);
    H[nd * di + di] = dot6(s, f);
    int j = i;
    while (r->links[j].parent >= 0) {
      transpose_force(kc->E[j], kc->r[j], f, f);
      j = r->links[j].parent;
      if (j == 0) {
        if (orc_dyn_floating(r))
          for (int k = 0; k < 6; ++k) H[nd * k + di] = H[nd * di + k] = f[k];
      } else if (r->links[j].joint == FSG_JOINT_REVOLUTE) {
        double sj[6] = {0, 0, 0, 0, 0, 0};
        normalized3(r->links[j].axis, sj);
        const int dj = orc_dyn_dof_index(r, j);
        H[nd * dj + di] = dot6(sj, f);
        H[nd * di + dj] = H[nd * dj + di];
      }
    }
  }
}

/* ---- bias_forces (RNEA, dynamics.hpp:118-155) ---------------------------- */
void orc_bias_forces(const fsg_robot* r, const fsg_joint_state* st, const orc_kcache* kc,
                     const double* g, double* c) {
  const int nb = r->n_links, nd = orc_dyn_n_dofs(r);
  double a[L][6], f[L][6];
  double rtg[3];
  mtv3(kc->R_world[0], g, rtg);
  a[0][0] = a[0][1] = a[0][2] = 0.0;
  for (int k = 0; k < 3; ++k) a[0][3 + k] = -rtg[k];
  for (int i = 0; i < nb; ++i) {
    const fsg_link* l = &r->links[i];
    if (i > 0) {
      apply_motion(kc->E[i], kc->r[i], a[l->parent], a[i]);
      if (l->joint == FSG_JOINT_REVOLUTE) {
        double s[6] = {0, 0, 0, 0, 0, 0}, cm[6];
        normalized3(l->axis, s);
        const double qd = st->v[orc_dyn_dof_index(r, i)];
        for (int k = 0; k < 6; ++k) s[k] = s[k] * qd;
        cross_motion(kc->v_body[i], s, cm);
        for (int k = 0; k < 6; ++k) a[i][k] = a[i][k] + cm[k];
      }
    }
    double ii[36], ia[6], iv[6], cf[6];
    orc_spatial_inertia(l->mass, l->com, l->inertia_com, ii);
    mv6(ii, a[i], ia);
    mv6(ii, kc->v_body[i], iv);
    cross_force(kc->v_body[i], iv, cf);
    for (int k = 0; k < 6; ++k) f[i][k] = ia[k] + cf[k];
  }
  memset(c, 0, (size_t)nd * sizeof(double));
  for (int i = nb - 1; i >= 0; --i) {
    const fsg_link* l = &r->links[i];
    if (i == 0) {
      if (orc_dyn_floating(r))
        for (int k = 0; k < 6; ++k) c[k] = f[0][k];
    } else {
      if (l->joint == FSG_JOINT_REVOLUTE) {
        double s[6] = {0, 0, 0, 0, 0, 0};
        normalized3(l->axis, s);
        c[orc_dyn_dof_index(r, i)] = dot6(s, f[i]);
      }
      double t[6];
      transpose_force(kc->E[i], kc->r[i], f[i], t);
      for (int k = 0; k < 6; ++k) f[l->parent][k] = f[l->parent][k] + t[k];
    }
  }
}

/* ---- internal_forces / joint_limit_forces (dynamics.hpp:160-198) --------- */
int orc_internal_forces(const fsg_robot* r, const fsg_joint_state* st, const double* act, double* tau) {
  const int nd = orc_dyn_n_dofs(r);
  int clamped = 0;
  memset(tau, 0, (size_t)nd * sizeof(double));
  for (int i = 1; i < r->n_links; ++i) {
    const fsg_link* l = &r->links[i];
    if (l->joint != FSG_JOINT_REVOLUTE) continue;
    const int di = orc_dyn_dof_index(r, i), ji = joint_index(r, i);
    double sigma = act[ji];
    if (fabs(sigma) > l->torque_limit) {
      sigma = sigma < -l->torque_limit ? -l->torque_limit : (sigma > l->torque_limit ? l->torque_limit : sigma);
      clamped = 1;
    }
    tau[di] = sigma - l->stiffness * (st->q[ji] - l->q_rest) - l->damping * st->v[di];
  }
  return clamped;
}
void orc_joint_limit_forces(const fsg_robot* r, const fsg_joint_state* st, double* tau) {
  const double k_limit = 50.0, c_limit = 0.5;
  memset(tau, 0, (size_t)orc_dyn_n_dofs(r) * sizeof(double));
  for (int i = 1; i < r->n_links; ++i) {
    const fsg_link* l = &r->links[i];
    if (l->joint != FSG_JOINT_REVOLUTE) continue;
    const int di = orc_dyn_dof_index(r, i), ji = joint_index(r, i);
    if (st->q[ji] > l->limit_hi)
      tau[di] = -k_limit * (st->q[ji] - l->limit_hi) - c_limit * fmax(st->v[di], 0.0);
    else if (st->q[ji] < l->limit_lo)
      tau[di] = -k_limit * (st->q[ji] - l->limit_lo) - c_limit * fmin(st->v[di], 0.0);
  }
}

/* ---- LLT (Cholesky) factor + solve ---------------------------------------- */
int orc_llt_solve(int n, const double* M, const double* b, double* x) {
  double Lm[ND * ND], y[ND];
  for (int j = 0; j < n; ++j) {
    double d = M[n * j + j];
    for (int k = 0; k < j; ++k) d -= Lm[n * j + k] * Lm[n * j + k];
    if (!(d > 0.0)) return 0;
    const double ljj = sqrt(d);
    Lm[n * j + j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      double s = M[n * i + j];
      for (int k = 0; k < j; ++k) s -= Lm[n * i + k] * Lm[n * j + k];
      Lm[n * i + j] = s / ljj;
    }
  }
  for (int i = 0; i < n; ++i) {
    double s = b[i];
    for (int k = 0; k < i; ++k) s -= Lm[n * i + k] * y[k];
    y[i] = s / Lm[n * i + i];
  }
  for (int i = n - 1; i >= 0; --i) { /* descending k, as the device kernels sum */
    double s = y[i];
    for (int k = n - 1; k > i; --k) s -= Lm[n * k + i] * x[k];
    x[i] = s / Lm[n * i + i];
  }
  return 1;
}

/* ---- forward_dynamics (dynamics.hpp:201-212) ------------------------------ */
int orc_forward_dynamics(const fsg_robot* r, const fsg_joint_state* st, const double* tau_int,
                         const double* tau_ext, const double* g, double* qdd) {
  const int nd = orc_dyn_n_dofs(r);
  orc_kcache kc;
  double M[ND * ND], c[ND], rhs[ND];
  orc_forward_kinematics(r, st, &kc);
  orc_mass_matrix(r, &kc, M);
  orc_bias_forces(r, st, &kc, g, c);
  for (int k = 0; k < nd; ++k) rhs[k] = (tau_int[k] + tau_ext[k]) - c[k];
  return orc_llt_solve(nd, M, rhs, qdd);
}

/* ---- accumulate_point_force / buoyancy_gravity_forces (dynamics.hpp:216-255) */
void orc_accumulate_point_force(const fsg_robot* r, const orc_kcache* kc, int link,
                                const double* p, const double* f, double* tau) {
  if (orc_dyn_floating(r)) {
    double d[3], m[3], t[3];
    for (int k = 0; k < 3; ++k) d[k] = p[k] - kc->p_world[0][k];
    cross3(d, f, m);
    mtv3(kc->R_world[0], m, t);
    for (int k = 0; k < 3; ++k) tau[k] = tau[k] + t[k];
    mtv3(kc->R_world[0], f, t);
    for (int k = 0; k < 3; ++k) tau[3 + k] = tau[3 + k] + t[k];
  }
  for (int j = link; j > 0; j = r->links[j].parent) {
    if (r->links[j].joint != FSG_JOINT_REVOLUTE) continue;
    double an[3], aw[3], d[3], m[3];
    normalized3(r->links[j].axis, an);
    mv3(kc->R_world[j], an, aw);
    for (int k = 0; k < 3; ++k) d[k] = p[k] - kc->p_world[j][k];
    cross3(aw, d, m);
    const int dj = orc_dyn_dof_index(r, j);
    tau[dj] = tau[dj] + dot3(m, f);
  }
}
void orc_buoyancy_gravity_forces(const fsg_robot* r, const orc_kcache* kc, double bladder_volume,
                                 double rho, const double* g, double* tau) {
  memset(tau, 0, (size_t)orc_dyn_n_dofs(r) * sizeof(double));
  for (int i = 0; i < r->n_links; ++i) {
    const fsg_link* l = &r->links[i];
    double t[3], p[3], f[3];
    mv3(kc->R_world[i], l->com, t);
    for (int k = 0; k < 3; ++k) p[k] = kc->p_world[i][k] + t[k], f[k] = l->mass * g[k];
    orc_accumulate_point_force(r, kc, i, p, f, tau);
    if (l->displaced_volume > 0.0) {
      const double s = -rho * l->displaced_volume;
      mv3(kc->R_world[i], l->volume_centroid, t);
      for (int k = 0; k < 3; ++k) p[k] = kc->p_world[i][k] + t[k], f[k] = s * g[k];
      orc_accumulate_point_force(r, kc, i, p, f, tau);
    }
  }
  if (bladder_volume > 0.0) {
    double t[3], p[3], f[3];
    const double s = -rho * bladder_volume;
    mv3(kc->R_world[0], r->bladder_centroid, t);
    for (int k = 0; k < 3; ++k) p[k] = kc->p_world[0][k] + t[k], f[k] = s * g[k];
    orc_accumulate_point_force(r, kc, 0, p, f, tau);
  }
}

/* ---- integrate (dynamics.hpp:259-289) ------------------------------------- */
int orc_integrate(const fsg_robot* r, fsg_joint_state* st, const double* act, const double* tau_ext,
                  double dt, int substeps, const double* g) {
  const int nd = orc_dyn_n_dofs(r);
  const double h = dt / substeps;
  int flags = 0;
  for (int s = 0; s < substeps; ++s) {
    double ti[ND], tl[ND], qdd[ND];
    if (orc_internal_forces(r, st, act, ti)) flags |= FSG_DYN_CLAMPED;
    orc_joint_limit_forces(r, st, tl);
    for (int k = 0; k < nd; ++k) ti[k] = ti[k] + tl[k];
    if (!orc_forward_dynamics(r, st, ti, tau_ext, g, qdd)) return flags | FSG_DYN_NOT_SPD;
    for (int k = 0; k < nd; ++k) st->qdd[k] = qdd[k], st->v[k] = st->v[k] + h * qdd[k];
    if (orc_dyn_floating(r)) {
      double R[9], t[3], w[3], dq[4], q[4];
      orc_quat_to_R(st->base_quat, R);
      mv3(R, st->v + 3, t);
      for (int k = 0; k < 3; ++k) st->base_pos[k] = st->base_pos[k] + h * t[k], w[k] = st->v[k] * h;
      orc_quat_exp(w, dq);
      quat_mul(st->base_quat, dq, q);
      quat_normalize(q);
      memcpy(st->base_quat, q, sizeof q);
    }
    for (int i = 1; i < r->n_links; ++i) {
      const fsg_link* l = &r->links[i];
      if (l->joint != FSG_JOINT_REVOLUTE) continue;
      const int di = orc_dyn_dof_index(r, i), ji = joint_index(r, i);
      st->q[ji] = st->q[ji] + h * st->v[di];
      if (st->q[ji] > l->limit_hi) {
        st->q[ji] = l->limit_hi;
        st->v[di] = fmin(st->v[di], 0.0);
      } else if (st->q[ji] < l->limit_lo) {
        st->q[ji] = l->limit_lo;
        st->v[di] = fmax(st->v[di], 0.0);
      }
    }
  }
  return flags;
}

/* session.hpp:169-175: hydro from the pre-step kinematics, then integrate */
int orc_robot_step(const fsg_robot* r, fsg_joint_state* st, double bladder_volume, const double* act,
                   const double* tau_ext, double rho, const double* g_hydro, double dt, int substeps,
                   const double* g) {
  const int nd = orc_dyn_n_dofs(r);
  double te[ND], hy[ND];
  const double zero[3] = {0, 0, 0};
  for (int k = 0; k < nd; ++k) te[k] = tau_ext ? tau_ext[k] : 0.0;
  if (g_hydro) {
    orc_kcache kc;
    orc_forward_kinematics(r, st, &kc);
    orc_buoyancy_gravity_forces(r, &kc, bladder_volume, rho, g_hydro, hy);
    for (int k = 0; k < nd; ++k) te[k] = te[k] + hy[k];
  }
  int flags = orc_integrate(r, st, act, te, dt, substeps, g ? g : zero);
  int finite = 1;
  for (int k = 0; k < nd; ++k) finite &= isfinite(st->v[k]);
  for (int k = 0; k < 3; ++k) finite &= isfinite(st->base_pos[k]);
  if (!finite) flags |= FSG_DYN_NONFINITE;
  return flags;
}

/* mechanical_energy (dynamics.hpp:292-303) */
double orc_mechanical_energy(const fsg_robot* r, const fsg_joint_state* st, const double* g) {
  orc_kcache kc;
  orc_forward_kinematics(r, st, &kc);
  double e = 0.0;
  for (int i = 0; i < r->n_links; ++i) {
    const fsg_link* l = &r->links[i];
    double ii[36], iv[6], t[3], cw[3];
    orc_spatial_inertia(l->mass, l->com, l->inertia_com, ii);
    mv6(ii, kc.v_body[i], iv);
    e += 0.5 * dot6(kc.v_body[i], iv);
    mv3(kc.R_world[i], l->com, t);
    for (int k = 0; k < 3; ++k) cw[k] = kc.p_world[i][k] + t[k];
    e -= l->mass * dot3(g, cw);
  }
  return e;
}

/* FK + BoneTransforms::of (skinning.hpp:90-99) into the fsg_body_pose layout */
void orc_dyn_pose(const fsg_robot* r, const fsg_joint_state* st, const double* rest_R,
                  const double* rest_p, fsg_body_pose* pose) {
  orc_kcache kc;
  memset(pose, 0, sizeof *pose);
  orc_forward_kinematics(r, st, &kc);
  for (int b = 0; b < r->n_links; ++b) {
    double rt[9], t[3];
    tr3(rest_R + 9 * b, rt);
    mm3(kc.R_world[b], rt, pose->bone_R[b]);
    mv3(pose->bone_R[b], rest_p + 3 * b, t);
    for (int k = 0; k < 3; ++k) pose->bone_t[b][k] = kc.p_world[b][k] - t[k];
    memcpy(pose->R_world[b], kc.R_world[b], 9 * sizeof(double));
    memcpy(pose->p_world[b], kc.p_world[b], 3 * sizeof(double));
    memcpy(pose->v_origin_world[b], kc.v_origin_world[b], 3 * sizeof(double));
    memcpy(pose->omega_world[b], kc.omega_world[b], 3 * sizeof(double));
  }
}
