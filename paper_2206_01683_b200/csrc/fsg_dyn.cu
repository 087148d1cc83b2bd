// fsg_dyn.cu -- articulated robot dynamics for a batch of envs on the device
// (SURVEY.md §8(f) #2): the robot half of CoupledSession::step
// (session.hpp:169-175) -- buoyancy_gravity_forces on the pre-step kinematics,
// then integrate() with its substeps -- for E robots of one skeleton, so the
// RL rollout loop's per-step robot work no longer round-trips through the
// host (tau_ext is produced on the device by the coupled step; the new pose
// feeds the device skinning).
//
// Mapping (one thread per env, fp64, --fmad=false, plain coefficient order):
//   forward_kinematics   dynamics.hpp:23-63    dk_fk
//   mass_matrix (CRBA)   dynamics.hpp:72-114   dk_crba  (X^T I X on the
//                        structured motion matrix: [E 0; -E S(r) E])
//   bias_forces (RNEA)   dynamics.hpp:118-155  dk_rnea
//   internal/limit       dynamics.hpp:160-198
//   forward_dynamics     dynamics.hpp:201-212  Cholesky (LLT) + 2 triangular solves
//   buoyancy_gravity     dynamics.hpp:216-255
//   integrate            dynamics.hpp:259-289  (quat_exp, types.hpp:71-79)
// The skeleton's invariants (normalised axes, dof/joint indices, link spatial
// inertias) are computed once on the host at create time with the same
// IEEE operations, and staged into shared memory by each block.  The robot
// math is tiny (nd <= 14) and latency-bound: a warp holds 32 envs.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/fsg.h"
#include "fsg_dyn_internal.h"

namespace {

constexpr int NL = FSG_DYN_MAX_LINKS;
constexpr int ND = FSG_DYN_MAX_DOFS;
constexpr int DYN_BLOCK = 32;

thread_local char g_dyn_err[512] = "";

int fail(int rc, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_dyn_err, sizeof g_dyn_err, fmt, ap);
  va_end(ap);
  return rc;
}

// the skeleton in the form the kernels read it
struct DynConst {
  int n_links, nd, nj, floating;
  int parent[NL], joint[NL], dof[NL], jidx[NL];
  double axis[NL][3];  // links[i].axis.normalized()
  double jorig[NL][3], jrot[NL][9];
  double I6[NL][36];   // spatial_inertia(mass, com, inertia_com), row-major
  double mass[NL], com[NL][3];
  double stiff[NL], damp[NL], q_rest[NL], lim_lo[NL], lim_hi[NL], tlim[NL];
  double dvol[NL], vcen[NL][3];
  double bl_centroid[3];
};

// ---- small algebra (identical operation order host and device) ----------
__host__ __device__ __forceinline__ void mv3(const double* A, const double* x, double* y) {
  const double y0 = A[0] * x[0] + A[1] * x[1] + A[2] * x[2];
  const double y1 = A[3] * x[0] + A[4] * x[1] + A[5] * x[2];
  const double y2 = A[6] * x[0] + A[7] * x[1] + A[8] * x[2];
  y[0] = y0, y[1] = y1, y[2] = y2;
}
__host__ __device__ __forceinline__ void mtv3(const double* A, const double* x, double* y) {
  const double y0 = A[0] * x[0] + A[3] * x[1] + A[6] * x[2];
  const double y1 = A[1] * x[0] + A[4] * x[1] + A[7] * x[2];
  const double y2 = A[2] * x[0] + A[5] * x[1] + A[8] * x[2];
  y[0] = y0, y[1] = y1, y[2] = y2;
}
__host__ __device__ __forceinline__ void mm3(const double* A, const double* B, double* C) {
  double t[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      t[3 * i + j] = A[3 * i] * B[j] + A[3 * i + 1] * B[3 + j] + A[3 * i + 2] * B[6 + j];
#pragma unroll
  for (int k = 0; k < 9; ++k) C[k] = t[k];
}
__host__ __device__ __forceinline__ void cross3(const double* a, const double* b, double* c) {
  const double c0 = a[1] * b[2] - a[2] * b[1];
  const double c1 = a[2] * b[0] - a[0] * b[2];
  const double c2 = a[0] * b[1] - a[1] * b[0];
  c[0] = c0, c[1] = c1, c[2] = c2;
}
__host__ __device__ __forceinline__ double dot3(const double* a, const double* b) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}
__host__ __device__ __forceinline__ void mv6(const double* A, const double* x, double* y) {
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) s += A[6 * i + k] * x[k];
    y[i] = s;
  }
}
// spatial.hpp:21-26 (E, r: the link's x_up)
__host__ __device__ __forceinline__ void apply_motion(const double* E, const double* r, const double* m,
                                             double* out) {
  double t[3], u[3], o[6];
  mv3(E, m, o);
  cross3(r, m, t);
  u[0] = m[3] - t[0], u[1] = m[4] - t[1], u[2] = m[5] - t[2];
  mv3(E, u, o + 3);
#pragma unroll
  for (int k = 0; k < 6; ++k) out[k] = o[k];
}
// spatial.hpp:37-42
__host__ __device__ __forceinline__ void transpose_force(const double* E, const double* r, const double* f,
                                                double* out) {
  double o[6], t[3];
  mtv3(E, f + 3, o + 3);
  mtv3(E, f, o);
  cross3(r, o + 3, t);
  o[0] = o[0] + t[0], o[1] = o[1] + t[1], o[2] = o[2] + t[2];
#pragma unroll
  for (int k = 0; k < 6; ++k) out[k] = o[k];
}

__host__ __device__ void quat_to_R(const double* q, double* R) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  const double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
  const double twx = tx * w, twy = ty * w, twz = tz * w;
  const double txx = tx * x, txy = ty * x, txz = tz * x;
  const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
  R[0] = 1.0 - (tyy + tzz), R[1] = txy - twz, R[2] = txz + twy;
  R[3] = txy + twz, R[4] = 1.0 - (txx + tzz), R[5] = tyz - twx;
  R[6] = txz - twy, R[7] = tyz + twx, R[8] = 1.0 - (txx + tyy);
}
// Eigen 3.4 AngleAxis::toRotationMatrix, unit axis
__host__ __device__ void angle_axis_R(double angle, const double* a, double* R) {
  double s, c;
  sincos(angle, &s, &c);
  const double sa0 = s * a[0], sa1 = s * a[1], sa2 = s * a[2];
  const double ca0 = (1.0 - c) * a[0], ca1 = (1.0 - c) * a[1], ca2 = (1.0 - c) * a[2];
  double t = ca0 * a[1];
  R[1] = t - sa2, R[3] = t + sa2;
  t = ca0 * a[2];
  R[2] = t + sa1, R[6] = t - sa1;
  t = ca1 * a[2];
  R[5] = t - sa0, R[7] = t + sa0;
  R[0] = ca0 * a[0] + c, R[4] = ca1 * a[1] + c, R[8] = ca2 * a[2] + c;
}
__host__ __device__ __forceinline__ void quat_normalize(double* q) {
  const double n = sqrt((q[1] * q[1] + q[3] * q[3]) + (q[2] * q[2] + q[0] * q[0]));
  q[0] = q[0] / n, q[1] = q[1] / n, q[2] = q[2] / n, q[3] = q[3] / n;
}

// KinematicsCache (dynamics.hpp:14-21) of one env, thread-private
struct KC {
  double E[NL][9], r[NL][3];
  double Rw[NL][9], pw[NL][3], vb[NL][6];
};

// forward_kinematics (dynamics.hpp:23-63)
__host__ __device__ void dk_fk(const DynConst& c, const fsg_joint_state& st, KC& k) {
  for (int i = 0; i < c.n_links; ++i) {
    if (i == 0) {
      quat_to_R(st.base_quat, k.Rw[0]);
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) k.E[0][3 * a + b] = k.Rw[0][3 * b + a];
#pragma unroll
      for (int a = 0; a < 3; ++a) k.pw[0][a] = st.base_pos[a], k.r[0][a] = st.base_pos[a];
#pragma unroll
      for (int a = 0; a < 6; ++a) k.vb[0][a] = c.floating ? st.v[a] : 0.0;
      continue;
    }
    double rj[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, rrel[9], t[3], qd = 0.0;
    const bool rev = c.joint[i] == FSG_JOINT_REVOLUTE;
    if (rev) {
      angle_axis_R(st.q[c.jidx[i]], c.axis[i], rj);
      qd = st.v[c.dof[i]];
    }
    mm3(c.jrot[i], rj, rrel);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) k.E[i][3 * a + b] = rrel[3 * b + a];
#pragma unroll
    for (int a = 0; a < 3; ++a) k.r[i][a] = c.jorig[i][a];
    const int pa = c.parent[i];
    mm3(k.Rw[pa], rrel, k.Rw[i]);
    mv3(k.Rw[pa], c.jorig[i], t);
#pragma unroll
    for (int a = 0; a < 3; ++a) k.pw[i][a] = k.pw[pa][a] + t[a];
    apply_motion(k.E[i], k.r[i], k.vb[pa], k.vb[i]);
    if (rev)
#pragma unroll
      for (int a = 0; a < 3; ++a) k.vb[i][a] = k.vb[i][a] + c.axis[i][a] * qd;
  }
}

// mass_matrix (dynamics.hpp:72-114).  ic[parent] += X^T ic X with
// X = [E 0; B E], B = -E S(r): the products skip X's zero block only (adding
// exact zeros), so each coefficient keeps the k = 0..5 summation order.
__host__ __device__ void dk_crba(const DynConst& c, const KC& k, double* H) {
  const int nb = c.n_links, nd = c.nd;
  double ic[NL][36];
  for (int i = 0; i < nb; ++i)
#pragma unroll
    for (int e = 0; e < 36; ++e) ic[i][e] = c.I6[i][e];
  for (int i = nb - 1; i >= 1; --i) {
    double X[36], T[36];
    {
      double S[9], ES[9];
      const double* r = k.r[i];
      S[0] = 0.0, S[1] = -r[2], S[2] = r[1], S[3] = r[2], S[4] = 0.0, S[5] = -r[0];
      S[6] = -r[1], S[7] = r[0], S[8] = 0.0;
      mm3(k.E[i], S, ES);
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          X[6 * a + b] = k.E[i][3 * a + b];
          X[6 * a + b + 3] = 0.0;
          X[6 * (a + 3) + b + 3] = k.E[i][3 * a + b];
          X[6 * (a + 3) + b] = -ES[3 * a + b];
        }
    }
#pragma unroll
    for (int a = 0; a < 6; ++a)
#pragma unroll
      for (int b = 0; b < 6; ++b) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < 6; ++q) s += X[6 * q + a] * ic[i][6 * q + b];
        T[6 * a + b] = s;
      }
    double* P = ic[c.parent[i]];
#pragma unroll
    for (int a = 0; a < 6; ++a)
#pragma unroll
      for (int b = 0; b < 6; ++b) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < 6; ++q) s += T[6 * a + q] * X[6 * q + b];
        P[6 * a + b] = P[6 * a + b] + s;
      }
  }
  for (int e = 0; e < nd * nd; ++e) H[e] = 0.0;
  if (c.floating)
    for (int a = 0; a < 6; ++a)
      for (int b = 0; b < 6; ++b) H[nd * a + b] = ic[0][6 * a + b];
  for (int i = 1; i < nb; ++i) {
    if (c.joint[i] != FSG_JOINT_REVOLUTE) continue;
    const int di = c.dof[i];
    const double s[6] = {c.axis[i][0], c.axis[i][1], c.axis[i][2], 0.0, 0.0, 0.0};
    double f[6];
    mv6(ic[i], s, f);
    {
      double d = 0.0;
#pragma unroll
      for (int q = 0; q < 6; ++q) d += s[q] * f[q];
      H[nd * di + di] = d;
    }
    int j = i;
    while (c.parent[j] >= 0) {
      transpose_force(k.E[j], k.r[j], f, f);
      j = c.parent[j];
      if (j == 0) {
        if (c.floating)
          for (int q = 0; q < 6; ++q) H[nd * q + di] = H[nd * di + q] = f[q];
      } else if (c.joint[j] == FSG_JOINT_REVOLUTE) {
        const double sj[6] = {c.axis[j][0], c.axis[j][1], c.axis[j][2], 0.0, 0.0, 0.0};
        double d = 0.0;
#pragma unroll
        for (int q = 0; q < 6; ++q) d += sj[q] * f[q];
        const int dj = c.dof[j];
        H[nd * dj + di] = d;
        H[nd * di + dj] = d;
      }
    }
  }
}

// bias_forces (dynamics.hpp:118-155)
__host__ __device__ void dk_rnea(const DynConst& c, const fsg_joint_state& st, const KC& k, const double* g,
                        double* cb) {
  const int nb = c.n_links;
  double a[NL][6], f[NL][6];
  {
    double rtg[3];
    mtv3(k.Rw[0], g, rtg);
    a[0][0] = a[0][1] = a[0][2] = 0.0;
    a[0][3] = -rtg[0], a[0][4] = -rtg[1], a[0][5] = -rtg[2];
  }
  for (int i = 0; i < nb; ++i) {
    if (i > 0) {
      apply_motion(k.E[i], k.r[i], a[c.parent[i]], a[i]);
      if (c.joint[i] == FSG_JOINT_REVOLUTE) {
        const double qd = st.v[c.dof[i]];
        const double m[6] = {c.axis[i][0] * qd, c.axis[i][1] * qd, c.axis[i][2] * qd, 0.0, 0.0, 0.0};
        // cross_motion(v, m) (spatial.hpp:55-60)
        const double* v = k.vb[i];
        double x0[3], x1[3], x2[3];
        cross3(v, m, x0);
        cross3(v, m + 3, x1);
        cross3(v + 3, m, x2);
        a[i][0] = a[i][0] + x0[0], a[i][1] = a[i][1] + x0[1], a[i][2] = a[i][2] + x0[2];
#pragma unroll
        for (int q = 0; q < 3; ++q) a[i][3 + q] = a[i][3 + q] + (x1[q] + x2[q]);
      }
    }
    double ia[6], iv[6], x0[3], x1[3], x2[3];
    mv6(c.I6[i], a[i], ia);
    mv6(c.I6[i], k.vb[i], iv);
    // cross_force(v, iv) (spatial.hpp:63-68)
    const double* v = k.vb[i];
    cross3(v, iv, x0);
    cross3(v + 3, iv + 3, x1);
    cross3(v, iv + 3, x2);
#pragma unroll
    for (int q = 0; q < 3; ++q) f[i][q] = ia[q] + (x0[q] + x1[q]), f[i][3 + q] = ia[3 + q] + x2[q];
  }
  for (int q = 0; q < c.nd; ++q) cb[q] = 0.0;
  for (int i = nb - 1; i >= 0; --i) {
    if (i == 0) {
      if (c.floating)
        for (int q = 0; q < 6; ++q) cb[q] = f[0][q];
      continue;
    }
    if (c.joint[i] == FSG_JOINT_REVOLUTE) {
      double d = 0.0;
#pragma unroll
      for (int q = 0; q < 3; ++q) d += c.axis[i][q] * f[i][q];
#pragma unroll
      for (int q = 3; q < 6; ++q) d += 0.0 * f[i][q];
      cb[c.dof[i]] = d;
    }
    double t[6];
    transpose_force(k.E[i], k.r[i], f[i], t);
    double* P = f[c.parent[i]];
#pragma unroll
    for (int q = 0; q < 6; ++q) P[q] = P[q] + t[q];
  }
}

// accumulate_point_force (dynamics.hpp:216-233)
__host__ __device__ void dk_point_force(const DynConst& c, const KC& k, int link, const double* p,
                               const double* f, double* tau) {
  if (c.floating) {
    double d[3], m[3], t[3];
    d[0] = p[0] - k.pw[0][0], d[1] = p[1] - k.pw[0][1], d[2] = p[2] - k.pw[0][2];
    cross3(d, f, m);
    mtv3(k.Rw[0], m, t);
    tau[0] = tau[0] + t[0], tau[1] = tau[1] + t[1], tau[2] = tau[2] + t[2];
    mtv3(k.Rw[0], f, t);
    tau[3] = tau[3] + t[0], tau[4] = tau[4] + t[1], tau[5] = tau[5] + t[2];
  }
  for (int j = link; j > 0; j = c.parent[j]) {
    if (c.joint[j] != FSG_JOINT_REVOLUTE) continue;
    double aw[3], d[3], m[3];
    mv3(k.Rw[j], c.axis[j], aw);
    d[0] = p[0] - k.pw[j][0], d[1] = p[1] - k.pw[j][1], d[2] = p[2] - k.pw[j][2];
    cross3(aw, d, m);
    tau[c.dof[j]] = tau[c.dof[j]] + dot3(m, f);
  }
}

// buoyancy_gravity_forces (dynamics.hpp:237-255), added onto tau
__host__ __device__ void dk_hydro(const DynConst& c, const KC& k, double bl_volume, double rho,
                         const double* g, double* tau) {
  double h[ND];
  for (int q = 0; q < c.nd; ++q) h[q] = 0.0;
  for (int i = 0; i < c.n_links; ++i) {
    double t[3], p[3], f[3];
    mv3(k.Rw[i], c.com[i], t);
#pragma unroll
    for (int q = 0; q < 3; ++q) p[q] = k.pw[i][q] + t[q], f[q] = c.mass[i] * g[q];
    dk_point_force(c, k, i, p, f, h);
    if (c.dvol[i] > 0.0) {
      const double s = -rho * c.dvol[i];
      mv3(k.Rw[i], c.vcen[i], t);
#pragma unroll
      for (int q = 0; q < 3; ++q) p[q] = k.pw[i][q] + t[q], f[q] = s * g[q];
      dk_point_force(c, k, i, p, f, h);
    }
  }
  if (bl_volume > 0.0) {
    double t[3], p[3], f[3];
    const double s = -rho * bl_volume;
    mv3(k.Rw[0], c.bl_centroid, t);
#pragma unroll
    for (int q = 0; q < 3; ++q) p[q] = k.pw[0][q] + t[q], f[q] = s * g[q];
    dk_point_force(c, k, 0, p, f, h);
  }
  for (int q = 0; q < c.nd; ++q) tau[q] = tau[q] + h[q];
}

// LLT (Cholesky) of M, then L y = b, L^T x = y; false when M is not SPD
__host__ __device__ bool dk_llt_solve(int n, double* M, const double* b, double* x) {
  for (int j = 0; j < n; ++j) {  // factor in place (lower triangle)
    double d = M[n * j + j];
    for (int q = 0; q < j; ++q) d -= M[n * j + q] * M[n * j + q];
    if (!(d > 0.0)) return false;
    const double ljj = sqrt(d);
    M[n * j + j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      double s = M[n * i + j];
      for (int q = 0; q < j; ++q) s -= M[n * i + q] * M[n * j + q];
      M[n * i + j] = s / ljj;
    }
  }
  double y[ND];
  for (int i = 0; i < n; ++i) {
    double s = b[i];
    for (int q = 0; q < i; ++q) s -= M[n * i + q] * y[q];
    y[i] = s / M[n * i + i];
  }
  for (int i = n - 1; i >= 0; --i) {  // (descending q: the order the warp kernel's
    double s = y[i];                    //  lanes accumulate as x[q] become known)
    for (int q = n - 1; q > i; --q) s -= M[n * q + i] * x[q];
    x[i] = s / M[n * i + i];
  }
  return true;
}

__device__ void load_const(DynConst& sc, const DynConst* gc) {
  const int n = (int)(sizeof(DynConst) / sizeof(int));
  const int* src = reinterpret_cast<const int*>(gc);
  int* dst = reinterpret_cast<int*>(&sc);
  for (int e = threadIdx.x; e < n; e += blockDim.x) dst[e] = src[e];
  __syncthreads();
}

// One robot step of one env (session.hpp:169-175 + dynamics.hpp:259-289);
// returns the FSG_DYN_* flags.
__host__ __device__ int dyn_env_step(const DynConst& c, fsg_joint_state& st, double bl_volume,
                                     const double* act, const double* tau_ext, double rho,
                                     int hydro, const double* gh, double dt, int substeps,
                                     const double* g) {
  const int nd = c.nd, nj = c.nj;
  double te[ND], sig[NL];
  for (int q = 0; q < nd; ++q) te[q] = tau_ext ? tau_ext[q] : 0.0;
  for (int q = 0; q < nj; ++q) sig[q] = act[q];
  KC k;
  if (hydro) {
    dk_fk(c, st, k);
    dk_hydro(c, k, bl_volume, rho, gh, te);
  }
  const double h = dt / substeps;
  int fl = 0;
  for (int s = 0; s < substeps; ++s) {
    // internal_forces + joint_limit_forces (dynamics.hpp:160-198)
    double ti[ND], tl[ND];
    for (int q = 0; q < nd; ++q) ti[q] = 0.0, tl[q] = 0.0;
    for (int i = 1; i < c.n_links; ++i) {
      if (c.joint[i] != FSG_JOINT_REVOLUTE) continue;
      const int di = c.dof[i], ji = c.jidx[i];
      double sigma = sig[ji];
      if (fabs(sigma) > c.tlim[i]) {
        sigma = fmin(fmax(sigma, -c.tlim[i]), c.tlim[i]);
        fl |= FSG_DYN_CLAMPED;
      }
      ti[di] = sigma - c.stiff[i] * (st.q[ji] - c.q_rest[i]) - c.damp[i] * st.v[di];
      if (st.q[ji] > c.lim_hi[i])
        tl[di] = -50.0 * (st.q[ji] - c.lim_hi[i]) - 0.5 * fmax(st.v[di], 0.0);
      else if (st.q[ji] < c.lim_lo[i])
        tl[di] = -50.0 * (st.q[ji] - c.lim_lo[i]) - 0.5 * fmin(st.v[di], 0.0);
    }
    // forward_dynamics (dynamics.hpp:201-212)
    double M[ND * ND], cb[ND], rhs[ND], qdd[ND];
    dk_fk(c, st, k);
    dk_crba(c, k, M);
    dk_rnea(c, st, k, g, cb);
    for (int q = 0; q < nd; ++q) rhs[q] = ((ti[q] + tl[q]) + te[q]) - cb[q];
    if (!dk_llt_solve(nd, M, rhs, qdd)) {
      fl |= FSG_DYN_NOT_SPD;
      break;
    }
    for (int q = 0; q < nd; ++q) st.qdd[q] = qdd[q], st.v[q] = st.v[q] + h * qdd[q];
    if (c.floating) {
      double R[9], t[3], w[3], dq[4], qn[4];
      quat_to_R(st.base_quat, R);
      mv3(R, st.v + 3, t);
#pragma unroll
      for (int q = 0; q < 3; ++q) st.base_pos[q] = st.base_pos[q] + h * t[q], w[q] = st.v[q] * h;
      // quat_exp (types.hpp:71-79)
      const double angle = sqrt(dot3(w, w));
      if (angle < 1e-12) {
        dq[0] = 1.0, dq[1] = 0.5 * w[0], dq[2] = 0.5 * w[1], dq[3] = 0.5 * w[2];
        quat_normalize(dq);
      } else {
        const double ax[3] = {w[0] / angle, w[1] / angle, w[2] / angle};
        double sh, ch;
        sincos(0.5 * angle, &sh, &ch);
        dq[0] = ch, dq[1] = sh * ax[0], dq[2] = sh * ax[1], dq[3] = sh * ax[2];
      }
      const double* a = st.base_quat;
      qn[0] = a[0] * dq[0] - a[1] * dq[1] - a[2] * dq[2] - a[3] * dq[3];
      qn[1] = a[0] * dq[1] + a[1] * dq[0] + a[2] * dq[3] - a[3] * dq[2];
      qn[2] = a[0] * dq[2] + a[2] * dq[0] + a[3] * dq[1] - a[1] * dq[3];
      qn[3] = a[0] * dq[3] + a[3] * dq[0] + a[1] * dq[2] - a[2] * dq[1];
      quat_normalize(qn);
#pragma unroll
      for (int q = 0; q < 4; ++q) st.base_quat[q] = qn[q];
    }
    for (int i = 1; i < c.n_links; ++i) {
      if (c.joint[i] != FSG_JOINT_REVOLUTE) continue;
      const int di = c.dof[i], ji = c.jidx[i];
      st.q[ji] = st.q[ji] + h * st.v[di];
      if (st.q[ji] > c.lim_hi[i]) {
        st.q[ji] = c.lim_hi[i];
        st.v[di] = fmin(st.v[di], 0.0);
      } else if (st.q[ji] < c.lim_lo[i]) {
        st.q[ji] = c.lim_lo[i];
        st.v[di] = fmax(st.v[di], 0.0);
      }
    }
  }
  bool finite = true;
  for (int q = 0; q < nd; ++q) finite &= isfinite(st.v[q]);
  for (int q = 0; q < 3; ++q) finite &= isfinite(st.base_pos[q]);
  if (!finite) fl |= FSG_DYN_NONFINITE;
  return fl;
}

__global__ void __launch_bounds__(DYN_BLOCK)
    k_dyn_step(const DynConst* __restrict__ gc, fsg_joint_state* __restrict__ states,
               const double* __restrict__ bladder, const double* __restrict__ act,
               const double* __restrict__ tau_ext, double rho, int hydro, double3 gh, double dt,
               int substeps, double3 gv, int* __restrict__ flags, int E,
               const double* const* __restrict__ tau_ptrs) {
  __shared__ DynConst c;
  load_const(c, gc);
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  fsg_joint_state st = states[e];
  const double ghv[3] = {gh.x, gh.y, gh.z}, gvv[3] = {gv.x, gv.y, gv.z};
  const double* te = tau_ptrs ? tau_ptrs[e] : (tau_ext ? tau_ext + (size_t)e * c.nd : nullptr);
  const int fl = dyn_env_step(c, st, bladder[e], act + (size_t)e * c.nj, te, rho, hydro, ghv, dt,
                              substeps, gvv);
  states[e] = st;
  if (flags) flags[e] = fl;
}

// ---- warp-per-env step (latency path for small batches) -------------------
// The same per-element arithmetic as dyn_env_step (so results are identical
// bit for bit), with the independent work spread over the lanes of one warp:
// per-link joint rotations, the 36 coefficients of each X^T I X product, the
// mass-matrix columns (one lane per revolute link), the per-link RNEA forces,
// and the rows of each Cholesky column.  The recursive chains (forward
// kinematics, RNEA sweeps, triangular solves) stay on lane 0; everything
// lives in shared memory.
constexpr int DYN_TWO_MAX = 256;  // envs up to which the warp kernel runs two warps per env
constexpr int DYN_WARPS = 3;  // 3 x ~13 KB warp workspaces + DynConst in 48 KB of static smem (12 links)

#ifdef FSG_DYN_TIMING  // dev builds only (scripts/build_variant.sh): per-phase clock64 of warp 0
__device__ unsigned long long g_dyn_t[8];
#define DYN_T(k)                                                        \
  do {                                                                  \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                          \
      const long long t_ = clock64();                                   \
      g_dyn_t[k] += (unsigned long long)(t_ - t_last);                  \
      t_last = t_;                                                      \
    }                                                                   \
  } while (0)
#else
#define DYN_T(k) \
  do {           \
  } while (0)
#endif

struct WarpWS {
  fsg_joint_state st;
  double rr[NL][9];  // r_rel of each link (link -> parent)
  KC k;  // E, r, Rw, pw, vb of every link
  double ic[NL][36];
  double X[36], T[36];
  double H[ND * ND];
  double a[NL][6], f[NL][6];
  double te[ND], tsum[ND], cb[ND], rhs[ND], y[ND], qdd[ND];
  double sig[NL];
  int ok, fl;
};

__device__ void wk_fk(const DynConst& c, WarpWS& w, int lane) {
  const fsg_joint_state& st = w.st;
  if (lane == 0) {
    quat_to_R(st.base_quat, w.k.Rw[0]);
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) w.k.E[0][3 * a + b] = w.k.Rw[0][3 * b + a];
    for (int a = 0; a < 3; ++a) w.k.pw[0][a] = st.base_pos[a], w.k.r[0][a] = st.base_pos[a];
    for (int a = 0; a < 6; ++a) w.k.vb[0][a] = c.floating ? st.v[a] : 0.0;
  } else if (lane < c.n_links) {
    const int i = lane;
    double rj[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    if (c.joint[i] == FSG_JOINT_REVOLUTE) angle_axis_R(st.q[c.jidx[i]], c.axis[i], rj);
    mm3(c.jrot[i], rj, w.rr[i]);
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) w.k.E[i][3 * a + b] = w.rr[i][3 * b + a];
    for (int a = 0; a < 3; ++a) w.k.r[i][a] = c.jorig[i][a];
  }
  __syncwarp();
  if (lane == 0) {
    for (int i = 1; i < c.n_links; ++i) {
      const int pa = c.parent[i];
      double t[3];
      mm3(w.k.Rw[pa], w.rr[i], w.k.Rw[i]);
      mv3(w.k.Rw[pa], c.jorig[i], t);
      for (int a = 0; a < 3; ++a) w.k.pw[i][a] = w.k.pw[pa][a] + t[a];
      apply_motion(w.k.E[i], w.k.r[i], w.k.vb[pa], w.k.vb[i]);
      if (c.joint[i] == FSG_JOINT_REVOLUTE) {
        const double qd = st.v[c.dof[i]];
        for (int a = 0; a < 3; ++a) w.k.vb[i][a] = w.k.vb[i][a] + c.axis[i][a] * qd;
      }
    }
  }
  __syncwarp();
}

__device__ void wk_crba(const DynConst& c, WarpWS& w, int lane) {
  const int nb = c.n_links, nd = c.nd;
  for (int e = lane; e < nb * 36; e += 32) w.ic[e / 36][e % 36] = c.I6[e / 36][e % 36];
  __syncwarp();
  for (int i = nb - 1; i >= 1; --i) {
    for (int e = lane; e < 36; e += 32) {  // X = [E 0; -E S(r) E]
      const int a = e / 6, b = e % 6;
      double x;
      if (a < 3) {
        x = b < 3 ? w.k.E[i][3 * a + b] : 0.0;
      } else if (b >= 3) {
        x = w.k.E[i][3 * (a - 3) + (b - 3)];
      } else {
        const double* r = w.k.r[i];
        const double S[9] = {0.0, -r[2], r[1], r[2], 0.0, -r[0], -r[1], r[0], 0.0};
        const double* A = w.k.E[i] + 3 * (a - 3);
        x = -(A[0] * S[b] + A[1] * S[3 + b] + A[2] * S[6 + b]);
      }
      w.X[e] = x;
    }
    __syncwarp();
    {  // T = X^T ic: element lane, and lane + 32 on lanes 0-3, as two
       // interleaved (independent) chains so the second hides behind the first
      const int e0 = lane, e1 = lane + 32 < 36 ? lane + 32 : lane;
      const int a0 = e0 / 6, b0 = e0 % 6, a1 = e1 / 6, b1 = e1 % 6;
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        s0 += w.X[6 * q + a0] * w.ic[i][6 * q + b0];
        s1 += w.X[6 * q + a1] * w.ic[i][6 * q + b1];
      }
      w.T[e0] = s0;
      if (e1 != e0) w.T[e1] = s1;
    }
    __syncwarp();
    double* P = w.ic[c.parent[i]];
    {  // ic[parent] += T X, the same two-chain split
      const int e0 = lane, e1 = lane + 32 < 36 ? lane + 32 : lane;
      const int a0 = e0 / 6, b0 = e0 % 6, a1 = e1 / 6, b1 = e1 % 6;
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        s0 += w.T[6 * a0 + q] * w.X[6 * q + b0];
        s1 += w.T[6 * a1 + q] * w.X[6 * q + b1];
      }
      const double p0 = P[e0] + s0;
      const double p1 = P[e1] + s1;
      P[e0] = p0;
      if (e1 != e0) P[e1] = p1;
    }
    __syncwarp();
  }
  for (int e = lane; e < nd * nd; e += 32) w.H[e] = 0.0;
  __syncwarp();
  if (c.floating)
    for (int e = lane; e < 36; e += 32) w.H[nd * (e / 6) + e % 6] = w.ic[0][e];
  const int i = lane;
  if (i >= 1 && i < nb && c.joint[i] == FSG_JOINT_REVOLUTE) {  // column of link i
    const int di = c.dof[i];
    const double s[6] = {c.axis[i][0], c.axis[i][1], c.axis[i][2], 0.0, 0.0, 0.0};
    double f[6];
    mv6(w.ic[i], s, f);
    double d = 0.0;
#pragma unroll
    for (int q = 0; q < 6; ++q) d += s[q] * f[q];
    w.H[nd * di + di] = d;
    int j = i;
    while (c.parent[j] >= 0) {
      transpose_force(w.k.E[j], w.k.r[j], f, f);
      j = c.parent[j];
      if (j == 0) {
        if (c.floating)
          for (int q = 0; q < 6; ++q) w.H[nd * q + di] = w.H[nd * di + q] = f[q];
      } else if (c.joint[j] == FSG_JOINT_REVOLUTE) {
        const double sj[6] = {c.axis[j][0], c.axis[j][1], c.axis[j][2], 0.0, 0.0, 0.0};
        double dd = 0.0;
#pragma unroll
        for (int q = 0; q < 6; ++q) dd += sj[q] * f[q];
        const int dj = c.dof[j];
        w.H[nd * dj + di] = dd;
        w.H[nd * di + dj] = dd;
      }
    }
  }
  __syncwarp();
}

__device__ void wk_rnea(const DynConst& c, WarpWS& w, int lane, const double* g) {
  const int nb = c.n_links;
  if (lane == 0) {
    double rtg[3];
    mtv3(w.k.Rw[0], g, rtg);
    w.a[0][0] = w.a[0][1] = w.a[0][2] = 0.0;
    w.a[0][3] = -rtg[0], w.a[0][4] = -rtg[1], w.a[0][5] = -rtg[2];
    for (int i = 1; i < nb; ++i) {
      apply_motion(w.k.E[i], w.k.r[i], w.a[c.parent[i]], w.a[i]);
      if (c.joint[i] == FSG_JOINT_REVOLUTE) {
        const double qd = w.st.v[c.dof[i]];
        const double m[6] = {c.axis[i][0] * qd, c.axis[i][1] * qd, c.axis[i][2] * qd, 0.0, 0.0, 0.0};
        const double* v = w.k.vb[i];
        double x0[3], x1[3], x2[3];
        cross3(v, m, x0);
        cross3(v, m + 3, x1);
        cross3(v + 3, m, x2);
        for (int q = 0; q < 3; ++q) w.a[i][q] = w.a[i][q] + x0[q];
        for (int q = 0; q < 3; ++q) w.a[i][3 + q] = w.a[i][3 + q] + (x1[q] + x2[q]);
      }
    }
  }
  __syncwarp();
  if (lane < nb) {
    const int i = lane;
    double ia[6], iv[6], x0[3], x1[3], x2[3];
    mv6(c.I6[i], w.a[i], ia);
    mv6(c.I6[i], w.k.vb[i], iv);
    const double* v = w.k.vb[i];
    cross3(v, iv, x0);
    cross3(v + 3, iv + 3, x1);
    cross3(v, iv + 3, x2);
    for (int q = 0; q < 3; ++q) w.f[i][q] = ia[q] + (x0[q] + x1[q]), w.f[i][3 + q] = ia[3 + q] + x2[q];
  }
  __syncwarp();
  if (lane == 0) {
    for (int q = 0; q < c.nd; ++q) w.cb[q] = 0.0;
    for (int i = nb - 1; i >= 0; --i) {
      if (i == 0) {
        if (c.floating)
          for (int q = 0; q < 6; ++q) w.cb[q] = w.f[0][q];
        continue;
      }
      if (c.joint[i] == FSG_JOINT_REVOLUTE) {
        double d = 0.0;
        for (int q = 0; q < 3; ++q) d += c.axis[i][q] * w.f[i][q];
        for (int q = 3; q < 6; ++q) d += 0.0 * w.f[i][q];
        w.cb[c.dof[i]] = d;
      }
      double t[6];
      transpose_force(w.k.E[i], w.k.r[i], w.f[i], t);
      double* P = w.f[c.parent[i]];
      for (int q = 0; q < 6; ++q) P[q] = P[q] + t[q];
    }
  }
  __syncwarp();
}

// Cholesky in place (as dk_llt_solve, element by element in the same order)
// with the rows of each column on lanes; the triangular solves on lane 0.
// (A register-resident variant -- rows in lane registers, right-looking
// rank-1 updates over shuffles -- measured slower: the solves' dependent
// divisions dominate either way.)
__device__ bool wk_llt_solve(WarpWS& w, int lane, int n) {
  double* M = w.H;
  // left-looking (a right-looking rank-1 variant, bit-identical, measured
  // slower: 67.4k vs 61.7k cycles per koi step -- the sqrt/division chain and
  // the extra barriers dominate)
  for (int j = 0; j < n; ++j) {
    if (lane == 0) {
      double d = M[n * j + j];
#pragma unroll 4
      for (int q = 0; q < j; ++q) d -= M[n * j + q] * M[n * j + q];
      w.ok = d > 0.0;
      if (w.ok) M[n * j + j] = sqrt(d);
    }
    __syncwarp();
    if (!w.ok) return false;
    const double ljj = M[n * j + j];
    const int i = j + 1 + lane;
    if (i < n) {
      double s = M[n * i + j];
#pragma unroll 4
      for (int q = 0; q < j; ++q) s -= M[n * i + q] * M[n * j + q];
      M[n * i + j] = s / ljj;
    }
    __syncwarp();
  }
  // triangular solves column by column: lane i keeps row i's running value
  // and subtracts L_ik y_k as soon as y_k is known -- for every row the same
  // operations in the same (ascending / descending k) order as the row-wise
  // dot products, so the result is bit-identical, but the dependent chain is
  // the n divisions instead of n^2/2 multiply-subtracts on one lane
  const unsigned full = 0xffffffffu;
  double b = lane < n ? w.rhs[lane] : 0.0;
  for (int k = 0; k < n; ++k) {
    const double yk = __shfl_sync(full, b, k) / M[n * k + k];
    if (lane == k) w.y[k] = yk;
    if (lane > k && lane < n) b = b - M[n * lane + k] * yk;
  }
  __syncwarp();
  b = lane < n ? w.y[lane] : 0.0;
  for (int k = n - 1; k >= 0; --k) {
    const double xk = __shfl_sync(full, b, k) / M[n * k + k];
    if (lane == k) w.qdd[k] = xk;
    if (lane < k) b = b - M[n * k + lane] * xk;
  }
  __syncwarp();
  return true;
}

/// Named barrier of an env's two warps (ids 1..DYN_WARPS; 0 is __syncthreads).
__device__ __forceinline__ void pair_sync(int wi) {
  // literal ids: a register id makes ptxas reserve all 16 barriers (one block per SM)
  static_assert(DYN_WARPS == 3, "one named barrier per env slot");
  if (wi == 0) asm volatile("bar.sync 1, 64;" ::: "memory");
  else if (wi == 1) asm volatile("bar.sync 2, 64;" ::: "memory");
  else asm volatile("bar.sync 3, 64;" ::: "memory");
}

/// TWO (latency-bound batches): two warps per env -- the main warp runs the
/// step, the helper warp runs RNEA (bias forces) while the main warp runs CRBA
/// (mass matrix): independent given the kinematics, disjoint workspace fields
/// (ic/X/T/H vs a/f/cb), the same arithmetic bit for bit (8 koi: 102.8 ->
/// 96.3 us per step).  Large batches keep one warp per env (the idle helper
/// warps cost throughput: 4096 envs 397 vs 582 us).
template <bool TWO>
__global__ void __launch_bounds__(64 * DYN_WARPS)
    k_dyn_step_warp(const DynConst* __restrict__ gc, fsg_joint_state* __restrict__ states,
                    const double* __restrict__ bladder, const double* __restrict__ act,
                    const double* __restrict__ tau_ext, double rho, int hydro, double3 gh,
                    double dt, int substeps, double3 gv, int* __restrict__ flags, int E,
                    const double* const* __restrict__ tau_ptrs) {
  __shared__ DynConst c;
  __shared__ WarpWS ws[DYN_WARPS];
  load_const(c, gc);
  const int lane = threadIdx.x & 31, wi = TWO ? threadIdx.x >> 6 : threadIdx.x >> 5;
  const bool helper = TWO && ((threadIdx.x >> 5) & 1);
  const int e = blockIdx.x * DYN_WARPS + wi;
  if (e >= E) return;  // (both warps of the env)
  WarpWS& w = ws[wi];
  const int nd = c.nd, nj = c.nj;
  if (helper) {  // RNEA of every substep, between the main warp's kinematics and its solve
    const double g[3] = {gv.x, gv.y, gv.z};
    for (int s = 0; s < substeps; ++s) {
      pair_sync(wi);  // kinematics of substep s ready (or the main warp stopped)
      if (w.ok < 0) break;
      wk_rnea(c, w, lane, g);
      pair_sync(wi);  // bias forces ready
    }
    return;
  }
#ifdef FSG_DYN_TIMING
  long long t_last = clock64();
#endif
  {
    const double* src = reinterpret_cast<const double*>(states + e);
    double* dst = reinterpret_cast<double*>(&w.st);
    for (int q = lane; q < (int)(sizeof(fsg_joint_state) / 8); q += 32) dst[q] = src[q];
  }
  {
    const double* te = tau_ptrs ? tau_ptrs[e] : (tau_ext ? tau_ext + (size_t)e * nd : nullptr);
    for (int q = lane; q < nd; q += 32) w.te[q] = te ? te[q] : 0.0;
  }
  for (int q = lane; q < nj; q += 32) w.sig[q] = act[(size_t)e * nj + q];
  if (lane == 0) w.fl = 0, w.ok = 0;  // (ok < 0: stop signal to the helper warp)
  __syncwarp();
  if (hydro) {
    wk_fk(c, w, lane);
    // buoyancy_gravity_forces on the pre-step kinematics (serial order, lane 0)
    if (lane == 0) {
      const double g[3] = {gh.x, gh.y, gh.z};
      dk_hydro(c, w.k, bladder[e], rho, g, w.te);
    }
    __syncwarp();
  }
  DYN_T(0);
  const double g[3] = {gv.x, gv.y, gv.z};
  const double h = dt / substeps;
  for (int s = 0; s < substeps; ++s) {
    // internal_forces + joint_limit_forces, one lane per link
    for (int q = lane; q < nd; q += 32) w.tsum[q] = 0.0 + 0.0;
    __syncwarp();
    bool clamped = false;
    if (lane >= 1 && lane < c.n_links && c.joint[lane] == FSG_JOINT_REVOLUTE) {
      const int i = lane, di = c.dof[i], ji = c.jidx[i];
      double sigma = w.sig[ji];
      if (fabs(sigma) > c.tlim[i]) {
        sigma = fmin(fmax(sigma, -c.tlim[i]), c.tlim[i]);
        clamped = true;
      }
      const double qi = w.st.q[ji], vi = w.st.v[di];
      const double ti = sigma - c.stiff[i] * (qi - c.q_rest[i]) - c.damp[i] * vi;
      double tl = 0.0;
      if (qi > c.lim_hi[i])
        tl = -50.0 * (qi - c.lim_hi[i]) - 0.5 * fmax(vi, 0.0);
      else if (qi < c.lim_lo[i])
        tl = -50.0 * (qi - c.lim_lo[i]) - 0.5 * fmin(vi, 0.0);
      w.tsum[di] = ti + tl;
    }
    if (__any_sync(0xffffffffu, clamped) && lane == 0) w.fl |= FSG_DYN_CLAMPED;
    DYN_T(1);
    // substep 0 after the hydrostatics: the kinematics of the unchanged
    // pre-step state are already in w (wk_fk writes w.k / w.rr from w.st only)
    if (s > 0 || !hydro) wk_fk(c, w, lane);
    if (TWO) pair_sync(wi);  // the helper warp starts RNEA
    DYN_T(2);
    wk_crba(c, w, lane);
    DYN_T(3);
    if (TWO) pair_sync(wi);  // RNEA done
    else wk_rnea(c, w, lane, g);
    for (int q = lane; q < nd; q += 32) w.rhs[q] = (w.tsum[q] + w.te[q]) - w.cb[q];
    __syncwarp();
    DYN_T(4);
    if (!wk_llt_solve(w, lane, nd)) {
      if (lane == 0) {
        w.fl |= FSG_DYN_NOT_SPD;
        w.ok = -1;  // the helper warp leaves at its next barrier
      }
      __syncwarp();
      if (TWO && s + 1 < substeps) pair_sync(wi);
      break;
    }
    DYN_T(5);
    if (lane == 0) {
      fsg_joint_state& st = w.st;
      for (int q = 0; q < nd; ++q) st.qdd[q] = w.qdd[q], st.v[q] = st.v[q] + h * w.qdd[q];
      if (c.floating) {
        double R[9], t[3], wv[3], dq[4], qn[4];
        quat_to_R(st.base_quat, R);
        mv3(R, st.v + 3, t);
        for (int q = 0; q < 3; ++q) st.base_pos[q] = st.base_pos[q] + h * t[q], wv[q] = st.v[q] * h;
        const double angle = sqrt(dot3(wv, wv));
        if (angle < 1e-12) {
          dq[0] = 1.0, dq[1] = 0.5 * wv[0], dq[2] = 0.5 * wv[1], dq[3] = 0.5 * wv[2];
          quat_normalize(dq);
        } else {
          const double ax[3] = {wv[0] / angle, wv[1] / angle, wv[2] / angle};
          double sh, ch;
          sincos(0.5 * angle, &sh, &ch);
          dq[0] = ch, dq[1] = sh * ax[0], dq[2] = sh * ax[1], dq[3] = sh * ax[2];
        }
        const double* a = st.base_quat;
        qn[0] = a[0] * dq[0] - a[1] * dq[1] - a[2] * dq[2] - a[3] * dq[3];
        qn[1] = a[0] * dq[1] + a[1] * dq[0] + a[2] * dq[3] - a[3] * dq[2];
        qn[2] = a[0] * dq[2] + a[2] * dq[0] + a[3] * dq[1] - a[1] * dq[3];
        qn[3] = a[0] * dq[3] + a[3] * dq[0] + a[1] * dq[2] - a[2] * dq[1];
        quat_normalize(qn);
        for (int q = 0; q < 4; ++q) st.base_quat[q] = qn[q];
      }
      for (int i = 1; i < c.n_links; ++i) {
        if (c.joint[i] != FSG_JOINT_REVOLUTE) continue;
        const int di = c.dof[i], ji = c.jidx[i];
        st.q[ji] = st.q[ji] + h * st.v[di];
        if (st.q[ji] > c.lim_hi[i]) {
          st.q[ji] = c.lim_hi[i];
          st.v[di] = fmin(st.v[di], 0.0);
        } else if (st.q[ji] < c.lim_lo[i]) {
          st.q[ji] = c.lim_lo[i];
          st.v[di] = fmax(st.v[di], 0.0);
        }
      }
    }
    __syncwarp();
    DYN_T(6);
  }
  if (lane == 0) {
    bool finite = true;
    for (int q = 0; q < nd; ++q) finite &= isfinite(w.st.v[q]);
    for (int q = 0; q < 3; ++q) finite &= isfinite(w.st.base_pos[q]);
    if (!finite) w.fl |= FSG_DYN_NONFINITE;
    if (flags) flags[e] = w.fl;
  }
  __syncwarp();
  {
    const double* src = reinterpret_cast<const double*>(&w.st);
    double* dst = reinterpret_cast<double*>(states + e);
    for (int q = lane; q < (int)(sizeof(fsg_joint_state) / 8); q += 32) dst[q] = src[q];
  }
}

__global__ void __launch_bounds__(DYN_BLOCK)
    k_dyn_mass(const DynConst* __restrict__ gc, const fsg_joint_state* __restrict__ states,
               double3 gv, double* __restrict__ M, double* __restrict__ bias, int E) {
  __shared__ DynConst c;
  load_const(c, gc);
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const fsg_joint_state st = states[e];
  KC k;
  dk_fk(c, st, k);
  const int nd = c.nd;
  double H[ND * ND], cb[ND];
  dk_crba(c, k, H);
  const double g[3] = {gv.x, gv.y, gv.z};
  dk_rnea(c, st, k, g, cb);
  if (M)
    for (int q = 0; q < nd * nd; ++q) M[(size_t)e * nd * nd + q] = H[q];
  if (bias)
    for (int q = 0; q < nd; ++q) bias[(size_t)e * nd + q] = cb[q];
}

// forward_kinematics + BoneTransforms::of (skinning.hpp:90-99) -> fsg_body_pose
__global__ void __launch_bounds__(DYN_BLOCK)
    k_dyn_pose(const DynConst* __restrict__ gc, const fsg_joint_state* __restrict__ states,
               const double* __restrict__ restR, const double* __restrict__ restp,
               char* __restrict__ poses, size_t stride, int E) {
  __shared__ DynConst c;
  load_const(c, gc);
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const fsg_joint_state st = states[e];
  KC k;
  dk_fk(c, st, k);
  fsg_body_pose& P = *reinterpret_cast<fsg_body_pose*>(poses + (size_t)e * stride);
  for (int b = 0; b < NL; ++b) {
    if (b >= c.n_links) {
      for (int q = 0; q < 9; ++q) P.bone_R[b][q] = 0.0, P.R_world[b][q] = 0.0;
      for (int q = 0; q < 3; ++q)
        P.bone_t[b][q] = P.p_world[b][q] = P.v_origin_world[b][q] = P.omega_world[b][q] = 0.0;
      continue;
    }
    double rt[9], bR[9], t[3], om[3], vo[3];
    for (int a = 0; a < 3; ++a)
      for (int q = 0; q < 3; ++q) rt[3 * a + q] = restR[9 * b + 3 * q + a];
    mm3(k.Rw[b], rt, bR);
    mv3(bR, restp + 3 * b, t);
    mv3(k.Rw[b], k.vb[b], om);
    mv3(k.Rw[b], k.vb[b] + 3, vo);
    for (int q = 0; q < 9; ++q) P.bone_R[b][q] = bR[q], P.R_world[b][q] = k.Rw[b][q];
    for (int q = 0; q < 3; ++q) {
      P.bone_t[b][q] = k.pw[b][q] - t[q];
      P.p_world[b][q] = k.pw[b][q];
      P.v_origin_world[b][q] = vo[q];
      P.omega_world[b][q] = om[q];
    }
  }
}

// RobotInstance::com_world (backend.hpp:24-33) of every env's current state:
// sum_i mass_i (p_world_i + R_world_i com_i) / sum_i mass_i, ascending links
// (Eigen's coefficient order), for the recentre trigger of session.hpp:181-193.
__global__ void __launch_bounds__(DYN_BLOCK)
    k_dyn_com(const DynConst* __restrict__ gc, const fsg_joint_state* __restrict__ states,
              double* __restrict__ com, int E) {
  __shared__ DynConst c;
  load_const(c, gc);
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  KC k;
  dk_fk(c, states[e], k);
  double w[3] = {0.0, 0.0, 0.0}, m = 0.0;
  for (int i = 0; i < c.n_links; ++i) {
    double rc[3];
    mv3(k.Rw[i], c.com[i], rc);
    for (int a = 0; a < 3; ++a) w[a] = w[a] + c.mass[i] * (k.pw[i][a] + rc[a]);
    m = m + c.mass[i];
  }
  for (int a = 0; a < 3; ++a) com[3 * e + a] = w[a] / m;
}

// ---- host ----------------------------------------------------------------
// Skeleton::validate (skeleton.hpp:95-118); messages follow the reference
// (links are named by index: fsg_link carries no name)
int validate(const fsg_robot& r) {
  if (r.n_links <= 0) return fail(FSG_EINPUT, "skeleton has no links");
  if (r.n_links > NL) return fail(FSG_EINPUT, "skeleton has %d links (max %d)", r.n_links, NL);
  if (r.links[0].parent != -1) return fail(FSG_EINPUT, "link 0 must be the root");
  if (r.links[0].joint == FSG_JOINT_REVOLUTE) return fail(FSG_EINPUT, "root joint must be free or fixed");
  for (int i = 0; i < r.n_links; ++i) {
    const fsg_link& l = r.links[i];
    if (l.joint < 0 || l.joint > 2) return fail(FSG_EINPUT, "link %d: unknown joint type", i);
    if (i == 0) continue;
    if (l.parent < 0 || l.parent >= i)
      return fail(FSG_EINPUT, "link %d: parent must precede it (tree order)", i);
    if (l.joint == FSG_JOINT_FREE) return fail(FSG_EINPUT, "link %d: only the root may be free", i);
    if (l.joint == FSG_JOINT_REVOLUTE && std::sqrt(dot3(l.axis, l.axis)) < 1e-12)
      return fail(FSG_EINPUT, "link %d: zero joint axis", i);
    if (l.limit_lo > l.limit_hi) return fail(FSG_EINPUT, "link %d: joint limits inverted", i);
  }
  for (int i = 0; i < r.n_links; ++i) {
    const fsg_link& l = r.links[i];
    if (!(l.mass > 0.0)) return fail(FSG_EINPUT, "link %d: mass must be positive", i);
    const double* I = l.inertia_com;
    double asym = 0.0, nrm = 0.0;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        const double d = I[3 * a + b] - I[3 * b + a];
        asym += d * d;
        nrm += I[3 * a + b] * I[3 * a + b];
      }
    if (std::sqrt(asym) > 1e-9 * (1.0 + std::sqrt(nrm)))
      return fail(FSG_EINPUT, "link %d: inertia tensor not symmetric", i);
    // positive definite <=> leading principal minors > 0 (Sylvester)
    const double m1 = I[0], m2 = I[0] * I[4] - I[1] * I[3];
    const double m3 = I[0] * (I[4] * I[8] - I[5] * I[7]) - I[1] * (I[3] * I[8] - I[5] * I[6]) +
                      I[2] * (I[3] * I[7] - I[4] * I[6]);
    if (!(m1 > 0.0 && m2 > 0.0 && m3 > 0.0))
      return fail(FSG_EINPUT, "link %d: inertia tensor not positive definite", i);
  }
  return FSG_OK;
}

void make_const(const fsg_robot& r, DynConst& c) {
  std::memset(&c, 0, sizeof c);
  c.n_links = r.n_links;
  c.floating = r.links[0].joint == FSG_JOINT_FREE;
  int nd = c.floating ? 6 : 0;
  for (int i = 0; i < r.n_links; ++i) {
    const fsg_link& l = r.links[i];
    c.parent[i] = l.parent;
    c.joint[i] = l.joint;
    c.dof[i] = i == 0 ? (c.floating ? 0 : -1) : -1;
    c.jidx[i] = -1;
    if (i > 0 && l.joint == FSG_JOINT_REVOLUTE) {
      c.dof[i] = nd;
      c.jidx[i] = nd - (c.floating ? 6 : 0);
      ++nd;
      const double n = std::sqrt(dot3(l.axis, l.axis));
      for (int a = 0; a < 3; ++a) c.axis[i][a] = l.axis[a] / n;
    }
    std::memcpy(c.jorig[i], l.joint_origin, sizeof c.jorig[i]);
    std::memcpy(c.jrot[i], l.joint_rotation, sizeof c.jrot[i]);
    c.mass[i] = l.mass;
    std::memcpy(c.com[i], l.com, sizeof c.com[i]);
    c.stiff[i] = l.stiffness, c.damp[i] = l.damping, c.q_rest[i] = l.q_rest;
    c.lim_lo[i] = l.limit_lo, c.lim_hi[i] = l.limit_hi, c.tlim[i] = l.torque_limit;
    c.dvol[i] = l.displaced_volume;
    std::memcpy(c.vcen[i], l.volume_centroid, sizeof c.vcen[i]);
    // spatial_inertia (spatial.hpp:72-80): [Ic + (m S) S^T, m S; m S^T, m 1]
    double S[9], St[9], mS[9], P[9];
    const double* p = l.com;
    S[0] = 0.0, S[1] = -p[2], S[2] = p[1], S[3] = p[2], S[4] = 0.0, S[5] = -p[0];
    S[6] = -p[1], S[7] = p[0], S[8] = 0.0;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) St[3 * a + b] = S[3 * b + a];
    for (int q = 0; q < 9; ++q) mS[q] = l.mass * S[q];
    mm3(mS, St, P);
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        c.I6[i][6 * a + b] = l.inertia_com[3 * a + b] + P[3 * a + b];
        c.I6[i][6 * a + b + 3] = mS[3 * a + b];
        c.I6[i][6 * (a + 3) + b] = l.mass * St[3 * a + b];
        c.I6[i][6 * (a + 3) + b + 3] = a == b ? l.mass : 0.0;
      }
  }
  c.nd = nd;
  c.nj = nd - (c.floating ? 6 : 0);
  std::memcpy(c.bl_centroid, r.bladder_centroid, sizeof c.bl_centroid);
}

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) return fail(FSG_ECUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
  } while (0)

}  // namespace

struct fsg_dyn {
  int dev = 0, E = 0;
  cudaStream_t s = nullptr;
  fsg_robot robot{};
  DynConst hc{};
  DynConst* d_c = nullptr;
  fsg_joint_state* d_state = nullptr;
  double* d_bladder = nullptr;
  std::vector<double> bladder;
  double *d_act = nullptr, *d_tau = nullptr, *d_rest = nullptr;
  int* d_flags = nullptr;
  double* d_M = nullptr;
  fsg_body_pose* d_pose = nullptr;
  // warp per env (latency) below FSG_DYN_WARP_MAX envs, else thread per env
  // (throughput); both compute the same arithmetic, bit for bit
  bool warp_kernel = true;
  bool rest_set = false;
};



namespace {
struct DevGuard {
  int prev = 0;
  explicit DevGuard(int d) {
    cudaGetDevice(&prev);
    cudaSetDevice(d);
  }
  ~DevGuard() { cudaSetDevice(prev); }
};
unsigned blocks(int E) { return (unsigned)((E + DYN_BLOCK - 1) / DYN_BLOCK); }
}  // namespace

// internal entry points for the batched coupled loop (fsg_session.cu)
namespace fsg {
int dyn_launch_step(fsg_dyn* d, const double* d_actuation, const double* d_tau_ext,
                    const double* const* d_tau_ptrs, double rho_fluid, const double* g_hydro,
                    double dt, int substeps, const double* gravity, int* d_flags, cudaStream_t s) {
  if (!d) return fail(FSG_EINPUT, "NULL handle");
  if (!d_actuation && d->hc.nj > 0) return fail(FSG_EINPUT, "actuation is NULL");
  if (substeps < 1) return fail(FSG_EINPUT, "substeps must be >= 1");
  if (!(dt > 0.0)) return fail(FSG_EINPUT, "dt must be positive");
  DevGuard g(d->dev);
  if (!s) s = d->s;
  const double3 gh = g_hydro ? make_double3(g_hydro[0], g_hydro[1], g_hydro[2]) : make_double3(0, 0, 0);
  const double3 gv = gravity ? make_double3(gravity[0], gravity[1], gravity[2]) : make_double3(0, 0, 0);
  const double* act = d_actuation ? d_actuation : d->d_act;
  const unsigned nblk = (unsigned)((d->E + DYN_WARPS - 1) / DYN_WARPS);
  if (d->warp_kernel && d->E <= DYN_TWO_MAX)
    k_dyn_step_warp<true><<<nblk, 64 * DYN_WARPS, 0, s>>>(
        d->d_c, d->d_state, d->d_bladder, act, d_tau_ext, rho_fluid, g_hydro ? 1 : 0, gh, dt,
        substeps, gv, d_flags, d->E, d_tau_ptrs);
  else if (d->warp_kernel)
    k_dyn_step_warp<false><<<nblk, 32 * DYN_WARPS, 0, s>>>(
        d->d_c, d->d_state, d->d_bladder, act, d_tau_ext, rho_fluid, g_hydro ? 1 : 0, gh, dt,
        substeps, gv, d_flags, d->E, d_tau_ptrs);
  else
    k_dyn_step<<<blocks(d->E), DYN_BLOCK, 0, s>>>(d->d_c, d->d_state, d->d_bladder, act, d_tau_ext,
                                                  rho_fluid, g_hydro ? 1 : 0, gh, dt, substeps, gv,
                                                  d_flags, d->E, d_tau_ptrs);
  CK(cudaGetLastError());
  return FSG_OK;
}

int dyn_launch_pose(fsg_dyn* d, void* dst, size_t stride, cudaStream_t s) {
  if (!d->rest_set) return fail(FSG_ESTATE, "fsg_dyn_set_rest has not been called");
  DevGuard g(d->dev);
  k_dyn_pose<<<blocks(d->E), DYN_BLOCK, 0, s>>>(d->d_c, d->d_state, d->d_rest, d->d_rest + 9 * NL,
                                                static_cast<char*>(dst), stride, d->E);
  CK(cudaGetLastError());
  return FSG_OK;
}

int dyn_upload_actuation(fsg_dyn* d, const double* act, cudaStream_t s, double** d_act) {
  DevGuard g(d->dev);
  CK(cudaStreamSynchronize(d->s));  // earlier fsg_dyn_* work on the handle's own stream
  if (d->hc.nj > 0)
    CK(cudaMemcpyAsync(d->d_act, act, sizeof(double) * d->E * d->hc.nj, cudaMemcpyHostToDevice, s));
  *d_act = d->d_act;
  return FSG_OK;
}

int dyn_launch_com(fsg_dyn* d, double* d_com, cudaStream_t s) {
  DevGuard g(d->dev);
  k_dyn_com<<<blocks(d->E), DYN_BLOCK, 0, s>>>(d->d_c, d->d_state, d_com, d->E);
  CK(cudaGetLastError());
  return FSG_OK;
}

int dyn_read_states(fsg_dyn* d, fsg_joint_state* out, int* flags, cudaStream_t s) {
  DevGuard g(d->dev);
  if (out)
    CK(cudaMemcpyAsync(out, d->d_state, sizeof(fsg_joint_state) * d->E, cudaMemcpyDeviceToHost, s));
  if (flags) CK(cudaMemcpyAsync(flags, d->d_flags, sizeof(int) * d->E, cudaMemcpyDeviceToHost, s));
  return FSG_OK;
}

int* dyn_flags(fsg_dyn* d) { return d->d_flags; }
const fsg_joint_state* dyn_states_dev(const fsg_dyn* d) { return d->d_state; }
int dyn_n_envs(const fsg_dyn* d) { return d->E; }
int dyn_n_links(const fsg_dyn* d) { return d->hc.n_links; }
bool dyn_rest_set(const fsg_dyn* d) { return d->rest_set; }
int dyn_device(const fsg_dyn* d) { return d->dev; }
}  // namespace fsg

extern "C" {

const char* fsg_dyn_last_error(void) { return g_dyn_err; }

#ifdef FSG_DYN_TIMING
int fsg_dyn_debug_timing(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_dyn_t, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(g_dyn_t, z, sizeof z);
  }
  return FSG_OK;
}
#endif

int fsg_dyn_create(const fsg_robot* robot, int n_envs, int device, fsg_dyn** out) {
  if (!out) return fail(FSG_EINPUT, "out is NULL");
  *out = nullptr;
  if (!robot) return fail(FSG_EINPUT, "robot is NULL");
  if (n_envs <= 0) return fail(FSG_EINPUT, "n_envs must be positive");
  int rc = validate(*robot);
  if (rc != FSG_OK) return rc;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return fail(FSG_ECUDA, "no CUDA device %d (the B200 path has no CPU fallback)", device);
  DevGuard g(device);
  auto* d = new fsg_dyn;
  d->dev = device;
  d->E = n_envs;
  d->robot = *robot;
  make_const(*robot, d->hc);
  {
    const char* env = std::getenv("FSG_DYN_WARP_MAX");
    const long wmax = env ? std::atol(env) : 2048;
    d->warp_kernel = n_envs <= wmax;
  }
  auto cleanup = [&](int r) {
    fsg_dyn_destroy(d);
    return r;
  };
  const int nd = d->hc.nd, nj = d->hc.nj;
  if (cudaStreamCreateWithFlags(&d->s, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&d->d_c, sizeof(DynConst)) != cudaSuccess ||
      cudaMalloc(&d->d_state, sizeof(fsg_joint_state) * n_envs) != cudaSuccess ||
      cudaMalloc(&d->d_bladder, sizeof(double) * n_envs) != cudaSuccess ||
      cudaMalloc(&d->d_act, sizeof(double) * n_envs * (nj > 0 ? nj : 1)) != cudaSuccess ||
      cudaMalloc(&d->d_tau, sizeof(double) * n_envs * nd) != cudaSuccess ||
      cudaMalloc(&d->d_rest, sizeof(double) * NL * 24) != cudaSuccess ||  // set_rest | poses scratch
      cudaMalloc(&d->d_flags, sizeof(int) * n_envs) != cudaSuccess ||
      cudaMalloc(&d->d_M, sizeof(double) * n_envs * (nd * nd + nd)) != cudaSuccess ||
      cudaMalloc(&d->d_pose, sizeof(fsg_body_pose) * n_envs) != cudaSuccess)
    return cleanup(fail(FSG_ECUDA, "device allocation failed: %s",
                        cudaGetErrorString(cudaGetLastError())));
  // JointState::zero (skeleton.hpp:144-150) with the robot's bladder
  std::vector<fsg_joint_state> z(n_envs);
  for (auto& s : z) {
    std::memset(&s, 0, sizeof s);
    s.base_quat[0] = 1.0;
  }
  d->bladder.assign(n_envs, robot->bladder_volume);
  if (cudaMemcpyAsync(d->d_c, &d->hc, sizeof(DynConst), cudaMemcpyHostToDevice, d->s) != cudaSuccess ||
      cudaMemcpyAsync(d->d_state, z.data(), sizeof(fsg_joint_state) * n_envs,
                      cudaMemcpyHostToDevice, d->s) != cudaSuccess ||
      cudaMemcpyAsync(d->d_bladder, d->bladder.data(), sizeof(double) * n_envs,
                      cudaMemcpyHostToDevice, d->s) != cudaSuccess ||
      cudaStreamSynchronize(d->s) != cudaSuccess)
    return cleanup(fail(FSG_ECUDA, "upload failed"));
  *out = d;
  return FSG_OK;
}

int fsg_dyn_destroy(fsg_dyn* d) {
  if (!d) return FSG_OK;
  DevGuard g(d->dev);
  if (d->s) cudaStreamSynchronize(d->s);
  cudaFree(d->d_c);
  cudaFree(d->d_state);
  cudaFree(d->d_bladder);
  cudaFree(d->d_act);
  cudaFree(d->d_tau);
  cudaFree(d->d_rest);
  cudaFree(d->d_flags);
  cudaFree(d->d_M);
  cudaFree(d->d_pose);
  if (d->s) cudaStreamDestroy(d->s);
  delete d;
  return FSG_OK;
}

int fsg_dyn_n_dofs(const fsg_dyn* d) { return d ? d->hc.nd : -1; }
int fsg_dyn_n_joints(const fsg_dyn* d) { return d ? d->hc.nj : -1; }

int fsg_dyn_set_state(fsg_dyn* d, const fsg_joint_state* states) {
  if (!d || !states) return fail(FSG_EINPUT, "NULL argument");
  DevGuard g(d->dev);
  CK(cudaMemcpyAsync(d->d_state, states, sizeof(fsg_joint_state) * d->E, cudaMemcpyHostToDevice, d->s));
  CK(cudaStreamSynchronize(d->s));
  return FSG_OK;
}

int fsg_dyn_get_state(fsg_dyn* d, fsg_joint_state* states) {
  if (!d || !states) return fail(FSG_EINPUT, "NULL argument");
  DevGuard g(d->dev);
  CK(cudaMemcpyAsync(states, d->d_state, sizeof(fsg_joint_state) * d->E, cudaMemcpyDeviceToHost, d->s));
  CK(cudaStreamSynchronize(d->s));
  return FSG_OK;
}

int fsg_dyn_change_bladder(fsg_dyn* d, const double* dv, double* volumes) {
  if (!d || !dv) return fail(FSG_EINPUT, "NULL argument");
  const fsg_robot& r = d->robot;
  for (int e = 0; e < d->E; ++e) {  // Bladder::apply_change (skeleton.hpp:48-51)
    const double step = std::min(std::max(dv[e], -r.bladder_rate_bound), r.bladder_rate_bound);
    d->bladder[e] = std::min(std::max(d->bladder[e] + step, r.bladder_volume_min), r.bladder_volume_max);
    if (volumes) volumes[e] = d->bladder[e];
  }
  DevGuard g(d->dev);
  CK(cudaMemcpyAsync(d->d_bladder, d->bladder.data(), sizeof(double) * d->E, cudaMemcpyHostToDevice, d->s));
  CK(cudaStreamSynchronize(d->s));
  return FSG_OK;
}

int fsg_dyn_step_device(fsg_dyn* d, const double* d_actuation, const double* d_tau_ext,
                        double rho_fluid, const double* g_hydro, double dt, int substeps,
                        const double* gravity, int* d_flags) {
  return fsg::dyn_launch_step(d, d_actuation, d_tau_ext, nullptr, rho_fluid, g_hydro, dt, substeps,
                              gravity, d_flags, nullptr);
}

int fsg_dyn_set_rest(fsg_dyn* d, const double* rest_R, const double* rest_p) {
  if (!d || !rest_R || !rest_p) return fail(FSG_EINPUT, "NULL argument");
  DevGuard g(d->dev);
  const int nl = d->hc.n_links;
  CK(cudaMemcpyAsync(d->d_rest, rest_R, sizeof(double) * 9 * nl, cudaMemcpyHostToDevice, d->s));
  CK(cudaMemcpyAsync(d->d_rest + 9 * NL, rest_p, sizeof(double) * 3 * nl, cudaMemcpyHostToDevice, d->s));
  CK(cudaStreamSynchronize(d->s));
  d->rest_set = true;
  return FSG_OK;
}

int fsg_dyn_step(fsg_dyn* d, const double* actuation, const double* tau_ext, double rho_fluid,
                 const double* g_hydro, double dt, int substeps, const double* gravity, int* flags) {
  if (!d) return fail(FSG_EINPUT, "NULL handle");
  if (!actuation && d->hc.nj > 0) return fail(FSG_EINPUT, "actuation is NULL");
  DevGuard g(d->dev);
  const int nd = d->hc.nd, nj = d->hc.nj;
  if (nj > 0)
    CK(cudaMemcpyAsync(d->d_act, actuation, sizeof(double) * d->E * nj, cudaMemcpyHostToDevice, d->s));
  if (tau_ext)
    CK(cudaMemcpyAsync(d->d_tau, tau_ext, sizeof(double) * d->E * nd, cudaMemcpyHostToDevice, d->s));
  int rc = fsg_dyn_step_device(d, d->d_act, tau_ext ? d->d_tau : nullptr, rho_fluid, g_hydro, dt,
                               substeps, gravity, d->d_flags);
  if (rc != FSG_OK) return rc;
  if (flags) CK(cudaMemcpyAsync(flags, d->d_flags, sizeof(int) * d->E, cudaMemcpyDeviceToHost, d->s));
  CK(cudaStreamSynchronize(d->s));
  return FSG_OK;
}

int fsg_dyn_mass_matrix(fsg_dyn* d, const double* gravity, double* M, double* bias) {
  if (!d) return fail(FSG_EINPUT, "NULL handle");
  DevGuard g(d->dev);
  const int nd = d->hc.nd;
  const double3 gv = gravity ? make_double3(gravity[0], gravity[1], gravity[2]) : make_double3(0, 0, 0);
  double* dM = d->d_M;
  double* dB = d->d_M + (size_t)d->E * nd * nd;
  k_dyn_mass<<<blocks(d->E), DYN_BLOCK, 0, d->s>>>(d->d_c, d->d_state, gv, dM, dB, d->E);
  CK(cudaGetLastError());
  if (M) CK(cudaMemcpyAsync(M, dM, sizeof(double) * d->E * nd * nd, cudaMemcpyDeviceToHost, d->s));
  if (bias) CK(cudaMemcpyAsync(bias, dB, sizeof(double) * d->E * nd, cudaMemcpyDeviceToHost, d->s));
  CK(cudaStreamSynchronize(d->s));
  return FSG_OK;
}

int fsg_dyn_poses(fsg_dyn* d, const double* rest_R, const double* rest_p, fsg_body_pose* poses) {
  if (!d || !rest_R || !rest_p || !poses) return fail(FSG_EINPUT, "NULL argument");
  DevGuard g(d->dev);
  const int nl = d->hc.n_links;
  // its own scratch: the rest pose fsg_dyn_set_rest gave the batched loop stays
  double* rs = d->d_rest + 12 * NL;
  CK(cudaMemcpyAsync(rs, rest_R, sizeof(double) * 9 * nl, cudaMemcpyHostToDevice, d->s));
  CK(cudaMemcpyAsync(rs + 9 * NL, rest_p, sizeof(double) * 3 * nl, cudaMemcpyHostToDevice, d->s));
  k_dyn_pose<<<blocks(d->E), DYN_BLOCK, 0, d->s>>>(d->d_c, d->d_state, rs, rs + 9 * NL,
                                                   reinterpret_cast<char*>(d->d_pose),
                                                   sizeof(fsg_body_pose), d->E);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(poses, d->d_pose, sizeof(fsg_body_pose) * d->E, cudaMemcpyDeviceToHost, d->s));
  CK(cudaStreamSynchronize(d->s));
  return FSG_OK;
}

}  // extern "C"
