/* fsg_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * fp64 restatement of the reference's hot path; see fsg_oracle.h.  Every
 * expression keeps the reference's evaluation order (Eigen's coefficient
 * order for the small vector algebra, see oracle/eigen_shim/Eigen/Dense) so
 * that it agrees with oracle/_ref bit-for-bit.  Compile with
 * -ffp-contract=off (oracle/Makefile).
 */
#include "fsg_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* lattice.hpp:17-38 */
const int ORC_EX[19] = {0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0};
const int ORC_EY[19] = {0, 0, 0, 1, -1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0, 1, -1, 1, -1};
const int ORC_EZ[19] = {0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1};
const double ORC_W[19] = {1.0 / 3.0,  1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0,
                          1.0 / 18.0, 1.0 / 18.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0,
                          1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0,
                          1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0};

static inline size_t cidx(const int d[3], int x, int y, int z) {
  return (size_t)x + (size_t)d[0] * ((size_t)y + (size_t)d[1] * (size_t)z);
}
static inline size_t ncells(const int d[3]) { return (size_t)d[0] * d[1] * d[2]; }
static inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* units.hpp:25-26 : tau = 3 nu dt/dx^2 + 1/2 */
double orc_tau(double dx, double dt, double nu) { return 3.0 * (nu * dt / (dx * dx)) + 0.5; }

/* lattice.hpp:41-45 */
double orc_equilibrium_dir(int i, double rho, const double u[3]) {
  const double eu = ORC_EX[i] * u[0] + ORC_EY[i] * u[1] + ORC_EZ[i] * u[2];
  const double u2 = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
  return ORC_W[i] * rho * (1.0 + 3.0 * eu + 4.5 * eu * eu - 1.5 * u2);
}

/* lattice.hpp:107-116 */
void orc_initialize(const int d[3], const double* rho, const double* u, double* f) {
  const size_t n = ncells(d);
  for (size_t c = 0; c < n; ++c)
    for (int i = 0; i < 19; ++i) f[i * n + c] = orc_equilibrium_dir(i, rho[c], u + 3 * c);
}

/* solver.hpp:25-51 */
int orc_macroscopic(const int d[3], const double* f, const double* F, double* rho_out,
                    double* u_out) {
  const size_t n = ncells(d);
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad)
  for (long long c = 0; c < (long long)n; ++c) {
    double rho = 0.0, mx = 0.0, my = 0.0, mz = 0.0;
    for (int i = 0; i < 19; ++i) {
      const double fi = f[i * n + c];
      rho += fi;
      mx += fi * ORC_EX[i];
      my += fi * ORC_EY[i];
      mz += fi * ORC_EZ[i];
    }
    rho_out[c] = rho;
    if (!(rho > 0.0)) {
      ++bad;
      u_out[3 * c] = u_out[3 * c + 1] = u_out[3 * c + 2] = 0.0;
      continue;
    }
    const double Fx = F ? F[3 * c] : 0.0, Fy = F ? F[3 * c + 1] : 0.0, Fz = F ? F[3 * c + 2] : 0.0;
    u_out[3 * c] = (mx + 0.5 * Fx) / rho;
    u_out[3 * c + 1] = (my + 0.5 * Fy) / rho;
    u_out[3 * c + 2] = (mz + 0.5 * Fz) / rho;
  }
  return bad;
}

/* solver.hpp:65-97 */
static void fix_cell(const int d[3], double* f, size_t n, int x, int y, int z) {
  const size_t c = cidx(d, x, y, z);
  const size_t cn = cidx(d, clampi(x, 1, d[0] - 2), clampi(y, 1, d[1] - 2), clampi(z, 1, d[2] - 2));
  for (int i = 0; i < 19; ++i) {
    const int sx = x - ORC_EX[i], sy = y - ORC_EY[i], sz = z - ORC_EZ[i];
    const int known = sx >= 0 && sx < d[0] && sy >= 0 && sy < d[1] && sz >= 0 && sz < d[2];
    if (!known) f[i * n + c] = f[i * n + cn];
  }
}
void orc_apply_open_boundary(const int d[3], double* f) {
  const size_t n = ncells(d);
#pragma omp parallel for schedule(static)
  for (int z = 0; z < d[2]; ++z)
    for (int y = 0; y < d[1]; ++y) {
      if (z == 0 || z == d[2] - 1 || y == 0 || y == d[1] - 1) {
        for (int x = 0; x < d[0]; ++x) fix_cell(d, f, n, x, y, z);
      } else {
        fix_cell(d, f, n, 0, y, z);
        fix_cell(d, f, n, d[0] - 1, y, z);
      }
    }
}

/* solver.hpp:103-178 (push streaming into fb, then open BC on fb) */
void orc_collide_and_stream(const int d[3], int periodic, double tau, const double* fa,
                            double* fb, const double* F, int* finite_out, double* min_f_out) {
  const int nx = d[0], ny = d[1], nz = d[2];
  const size_t n = ncells(d);
  const double omega = 1.0 / tau;
  const double guo_pref = 1.0 - 0.5 * omega;
  long long off[19];
  for (int i = 0; i < 19; ++i) off[i] = ORC_EX[i] + (long long)nx * (ORC_EY[i] + (long long)ny * ORC_EZ[i]);
  double min_f = DBL_MAX;
  int finite = 1;
#pragma omp parallel for schedule(static) reduction(min : min_f) reduction(&& : finite)
  for (int z = 0; z < nz; ++z) {
    for (int y = 0; y < ny; ++y) {
      const int row_interior = z > 0 && z < nz - 1 && y > 0 && y < ny - 1;
      for (int x = 0; x < nx; ++x) {
        const size_t c = cidx(d, x, y, z);
        double fi[19];
        double rho = 0.0, mx = 0.0, my = 0.0, mz = 0.0;
        for (int i = 0; i < 19; ++i) {
          fi[i] = fa[i * n + c];
          rho += fi[i];
          mx += fi[i] * ORC_EX[i];
          my += fi[i] * ORC_EY[i];
          mz += fi[i] * ORC_EZ[i];
        }
        const double Fx = F[3 * c], Fy = F[3 * c + 1], Fz = F[3 * c + 2];
        const double inv_rho = 1.0 / rho;
        const double ux = (mx + 0.5 * Fx) * inv_rho;
        const double uy = (my + 0.5 * Fy) * inv_rho;
        const double uz = (mz + 0.5 * Fz) * inv_rho;
        const double u2 = ux * ux + uy * uy + uz * uz;
        if (!isfinite(rho + u2)) finite = 0;
        const int interior = row_interior && x > 0 && x < nx - 1;
        for (int i = 0; i < 19; ++i) {
          const double eu = ORC_EX[i] * ux + ORC_EY[i] * uy + ORC_EZ[i] * uz;
          const double feq = ORC_W[i] * rho * (1.0 + 3.0 * eu + 4.5 * eu * eu - 1.5 * u2);
          const double sx = 3.0 * (ORC_EX[i] - ux) + 9.0 * eu * ORC_EX[i];
          const double sy = 3.0 * (ORC_EY[i] - uy) + 9.0 * eu * ORC_EY[i];
          const double sz = 3.0 * (ORC_EZ[i] - uz) + 9.0 * eu * ORC_EZ[i];
          const double src = guo_pref * ORC_W[i] * (sx * Fx + sy * Fy + sz * Fz);
          const double post = fi[i] - omega * (fi[i] - feq) + src;
          if (post < min_f) min_f = post;
          if (interior) {
            fb[i * n + c + off[i]] = post;
          } else {
            int tx = x + ORC_EX[i], ty = y + ORC_EY[i], tz = z + ORC_EZ[i];
            if (periodic) {
              tx = (tx + nx) % nx;
              ty = (ty + ny) % ny;
              tz = (tz + nz) % nz;
            } else if (tx < 0 || tx >= nx || ty < 0 || ty >= ny || tz < 0 || tz >= nz) {
              continue;
            }
            fb[i * n + cidx(d, tx, ty, tz)] = post;
          }
        }
      }
    }
  }
  if (!periodic) orc_apply_open_boundary(d, fb);
  *finite_out = finite;
  *min_f_out = min_f;
}

/* solver.hpp:181-200 */
double orc_total_mass(const int d[3], const double* f) {
  const size_t total = ncells(d) * 19;
  double s = 0.0;
  for (size_t k = 0; k < total; ++k) s += f[k];
  return s;
}
void orc_total_momentum(const int d[3], const double* f, double p[3]) {
  const size_t n = ncells(d);
  p[0] = p[1] = p[2] = 0.0;
  for (int i = 0; i < 19; ++i) {
    double s = 0.0;
    const double* fi = f + (size_t)i * n;
    for (size_t c = 0; c < n; ++c) s += fi[c];
    p[0] = p[0] + s * (double)ORC_EX[i];
    p[1] = p[1] + s * (double)ORC_EY[i];
    p[2] = p[2] + s * (double)ORC_EZ[i];
  }
}

/* kernel.hpp:22-33 */
double orc_phi(int kernel, double r) {
  const double a = fabs(r);
  if (kernel == 0) {
    if (a >= 2.0) return 0.0;
    if (a <= 1.0) return 0.125 * (3.0 - 2.0 * a + sqrt(1.0 + 4.0 * a - 4.0 * a * a));
    return 0.125 * (5.0 - 2.0 * a - sqrt(-7.0 + 12.0 * a - 4.0 * a * a));
  }
  if (a <= 0.5) return (1.0 + sqrt(1.0 - 3.0 * r * r)) / 3.0;
  if (a <= 1.5) return (5.0 - 3.0 * a - sqrt(-3.0 * (1.0 - a) * (1.0 - a) + 1.0)) / 6.0;
  return 0.0;
}
/* kernel.hpp:36-40 */
void orc_range(int kernel, double x, int* lo, int* hi) {
  const double half = 0.5 * (kernel == 0 ? 4 : 3);
  *lo = (int)ceil(x - half);
  *hi = (int)floor(x + half);
}
/* coupling.hpp:18-24 */
int orc_marker_in_bounds(int kernel, const int d[3], const double x[3]) {
  const double margin = 0.5 * (kernel == 0 ? 4 : 3);
  for (int a = 0; a < 3; ++a)
    if (x[a] < margin || x[a] > d[a] - 1 - margin) return 0;
  return 1;
}
static inline int imax(int a, int b) { return a > b ? a : b; }
static inline int imin(int a, int b) { return a < b ? a : b; }

/* coupling.hpp:27-48 */
void orc_interpolate(int kernel, const int d[3], const double* uf, const double x[3],
                     double out[3]) {
  int xlo, xhi, ylo, yhi, zlo, zhi;
  orc_range(kernel, x[0], &xlo, &xhi);
  orc_range(kernel, x[1], &ylo, &yhi);
  orc_range(kernel, x[2], &zlo, &zhi);
  double u0 = 0.0, u1 = 0.0, u2 = 0.0;
  for (int k = imax(zlo, 0); k <= imin(zhi, d[2] - 1); ++k) {
    const double wz = orc_phi(kernel, k - x[2]);
    for (int j = imax(ylo, 0); j <= imin(yhi, d[1] - 1); ++j) {
      const double wyz = wz * orc_phi(kernel, j - x[1]);
      for (int i = imax(xlo, 0); i <= imin(xhi, d[0] - 1); ++i) {
        const double w = wyz * orc_phi(kernel, i - x[0]);
        const size_t c = cidx(d, i, j, k);
        u0 = u0 + w * uf[3 * c];
        u1 = u1 + w * uf[3 * c + 1];
        u2 = u2 + w * uf[3 * c + 2];
      }
    }
  }
  out[0] = u0;
  out[1] = u1;
  out[2] = u2;
}

/* coupling.hpp:52-71 */
void orc_spread(int kernel, const int d[3], double* F, const double x[3], const double f[3]) {
  int xlo, xhi, ylo, yhi, zlo, zhi;
  orc_range(kernel, x[0], &xlo, &xhi);
  orc_range(kernel, x[1], &ylo, &yhi);
  orc_range(kernel, x[2], &zlo, &zhi);
  for (int k = imax(zlo, 0); k <= imin(zhi, d[2] - 1); ++k) {
    const double wz = orc_phi(kernel, k - x[2]);
    for (int j = imax(ylo, 0); j <= imin(yhi, d[1] - 1); ++j) {
      const double wyz = wz * orc_phi(kernel, j - x[1]);
      for (int i = imax(xlo, 0); i <= imin(xhi, d[0] - 1); ++i) {
        const double w = wyz * orc_phi(kernel, i - x[0]);
        const size_t c = cidx(d, i, j, k);
        F[3 * c] = F[3 * c] + w * f[0];
        F[3 * c + 1] = F[3 * c + 1] + w * f[1];
        F[3 * c + 2] = F[3 * c + 2] + w * f[2];
      }
    }
  }
}

static inline double dot3(const double a[3], const double b[3]) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}
static inline void cross3(const double a[3], const double b[3], double r[3]) {
  r[0] = a[1] * b[2] - a[2] * b[1];
  r[1] = a[2] * b[0] - a[0] * b[2];
  r[2] = a[0] * b[1] - a[1] * b[0];
}
/* row-major R: r = R v, Eigen coefficient order */
static inline void matvec(const double R[9], const double v[3], double r[3]) {
  for (int i = 0; i < 3; ++i) r[i] = R[3 * i] * v[0] + R[3 * i + 1] * v[1] + R[3 * i + 2] * v[2];
}
/* r = R^T v */
static inline void matTvec(const double R[9], const double v[3], double r[3]) {
  for (int i = 0; i < 3; ++i) r[i] = R[i] * v[0] + R[3 + i] * v[1] + R[6 + i] * v[2];
}

/* coupling.hpp:80-85 */
void orc_direct_forcing(const double ub[3], const double uf[3], const double n[3], double rho,
                        double area, double h, double dt, int wall, double out[3]) {
  double du[3] = {ub[0] - uf[0], ub[1] - uf[1], ub[2] - uf[2]};
  if (wall == 0) {
    const double s = dot3(du, n);
    du[0] = s * n[0];
    du[1] = s * n[1];
    du[2] = s * n[2];
  }
  const double k = rho * area * h / dt;
  out[0] = k * du[0];
  out[1] = k * du[1];
  out[2] = k * du[2];
}

/* frame.hpp:21 (Eigen Quaternion::toRotationMatrix), frame.hpp:48-50 */
void orc_frame_consts_of(const orc_frame_state* fs, orc_frame_consts* fc) {
  const double w = fs->q[0], x = fs->q[1], y = fs->q[2], z = fs->q[3];
  const double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
  const double twx = tx * w, twy = ty * w, twz = tz * w;
  const double txx = tx * x, txy = ty * x, txz = tz * x;
  const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
  double* R = fc->R;
  R[0] = 1.0 - (tyy + tzz);
  R[1] = txy - twz;
  R[2] = txz + twy;
  R[3] = txy + twz;
  R[4] = 1.0 - (txx + tzz);
  R[5] = tyz - twx;
  R[6] = txz - twy;
  R[7] = tyz + twx;
  R[8] = 1.0 - (txx + tyy);
  matTvec(R, fs->pdd, fc->a0);
  matTvec(R, fs->omega, fc->omega_f);
  matTvec(R, fs->alpha, fc->alpha_f);
}

/* frame.hpp:47-53 : -(R^T pdd) - a' x x - w' x (w' x x) - 2 w' x u */
void orc_virtual_force(const orc_frame_consts* fc, const double x[3], const double u[3],
                       double out[3]) {
  double ax[3], wx[3], wwx[3], wu[3];
  cross3(fc->alpha_f, x, ax);
  cross3(fc->omega_f, x, wx);
  cross3(fc->omega_f, wx, wwx);
  cross3(fc->omega_f, u, wu);
  for (int k = 0; k < 3; ++k) out[k] = -fc->a0[k] - ax[k] - wwx[k] - 2.0 * wu[k];
}

/* frame.hpp:132-154 */
void orc_recenter(const int d[3], double dx, const double* src, double* dst, const int shift[3],
                  orc_frame_state* fs) {
  const size_t n = ncells(d);
#pragma omp parallel for schedule(static)
  for (int z = 0; z < d[2]; ++z)
    for (int y = 0; y < d[1]; ++y)
      for (int x = 0; x < d[0]; ++x) {
        const int sx = clampi(x + shift[0], 0, d[0] - 1);
        const int sy = clampi(y + shift[1], 0, d[1] - 1);
        const int sz = clampi(z + shift[2], 0, d[2] - 1);
        const size_t cd = cidx(d, x, y, z), cs = cidx(d, sx, sy, sz);
        for (int i = 0; i < 19; ++i) dst[i * n + cd] = src[i * n + cs];
      }
  if (fs) {
    orc_frame_consts fc;
    orc_frame_consts_of(fs, &fc);
    const double off[3] = {shift[0] * dx, shift[1] * dx, shift[2] * dx};
    double r[3];
    matvec(fc.R, off, r);
    for (int k = 0; k < 3; ++k) fs->p[k] = fs->p[k] + r[k];
  }
}

/* ------------------------------------------------------------ session --- */
struct orc_session {
  int d[3];
  double dx, dt, rho_phys, nu, tau;
  int periodic, kernel, wall, frame_mode;
  double *fa, *fb, *F, *rho, *u;
  orc_frame_state fs;
};

orc_session* orc_session_create(const int d[3], double dx, double dt, double rho, double nu,
                                int periodic, int kernel, int wall, int frame_mode) {
  orc_session* s = (orc_session*)calloc(1, sizeof *s);
  memcpy(s->d, d, sizeof s->d);
  s->dx = dx;
  s->dt = dt;
  s->rho_phys = rho;
  s->nu = nu;
  s->tau = orc_tau(dx, dt, nu);
  s->periodic = periodic;
  s->kernel = kernel;
  s->wall = wall;
  s->frame_mode = frame_mode;
  const size_t n = ncells(d);
  s->fa = (double*)malloc(sizeof(double) * 19 * n);
  s->fb = (double*)malloc(sizeof(double) * 19 * n);
  s->F = (double*)calloc(3 * n, sizeof(double));
  s->rho = (double*)malloc(sizeof(double) * n);
  s->u = (double*)calloc(3 * n, sizeof(double));
  for (int i = 0; i < 19; ++i)
    for (size_t c = 0; c < n; ++c) s->fa[i * n + c] = ORC_W[i];
  for (size_t c = 0; c < n; ++c) s->rho[c] = 1.0;
  s->fs.q[0] = 1.0;
  return s;
}
void orc_session_destroy(orc_session* s) {
  if (!s) return;
  free(s->fa);
  free(s->fb);
  free(s->F);
  free(s->rho);
  free(s->u);
  free(s);
}
double* orc_session_f(orc_session* s) { return s->fa; }
double* orc_session_force(orc_session* s) { return s->F; }
double* orc_session_rho(orc_session* s) { return s->rho; }
double* orc_session_u(orc_session* s) { return s->u; }
void orc_session_set_frame(orc_session* s, const orc_frame_state* fs) { s->fs = *fs; }
void orc_session_get_frame(orc_session* s, orc_frame_state* fs) { *fs = s->fs; }

/* session.hpp:94-166 (fluid half; caller supplies world-frame markers) */
int orc_session_step(orc_session* s, int n_bodies, const int64_t* off, const double* points,
                     const double* velocities, const double* normals, const double* areas,
                     double* force_world, int* valid, double* stats, int* finite, double* min_f) {
  const int* d = s->d;
  const size_t n = ncells(d);
  const double dt = s->dt, dx = s->dx;
  orc_frame_consts fc;
  orc_frame_consts_of(&s->fs, &fc);
  memset(s->F, 0, sizeof(double) * 3 * n);
  const int nonpos = orc_macroscopic(d, s->fa, NULL, s->rho, s->u);
  const double half_d[3] = {0.5 * (d[0] - 1), 0.5 * (d[1] - 1), 0.5 * (d[2] - 1)};

  for (int b = 0; b < n_bodies; ++b) {
    const long long m0 = off[b], m1 = off[b + 1];
#pragma omp parallel for schedule(static)
    for (long long g = m0; g < m1; ++g) {
      double xw[3], xf[3], xl[3];
      for (int k = 0; k < 3; ++k) xw[k] = points[3 * g + k] - s->fs.p[k];
      matTvec(fc.R, xw, xf); /* world_to_frame_point, frame.hpp:24-26 */
      for (int k = 0; k < 3; ++k) xl[k] = xf[k] / dx + half_d[k]; /* session.hpp:82-85 */
      valid[g] = 0;
      force_world[3 * g] = force_world[3 * g + 1] = force_world[3 * g + 2] = 0.0;
      if (!orc_marker_in_bounds(s->kernel, d, xl)) continue;
      valid[g] = 1;
      double ui[3], uf[3], vw[3], vf[3], wx[3], ub[3], nf[3], fl[3];
      orc_interpolate(s->kernel, d, s->u, xl, ui);
      const double v2p = dx / dt; /* units.hpp:31 */
      for (int k = 0; k < 3; ++k) uf[k] = ui[k] * v2p;
      /* body_velocity_to_frame, frame.hpp:39-42 */
      for (int k = 0; k < 3; ++k) vw[k] = velocities[3 * g + k] - s->fs.pd[k];
      matTvec(fc.R, vw, vf);
      cross3(fc.omega_f, xf, wx);
      for (int k = 0; k < 3; ++k) ub[k] = vf[k] - wx[k];
      matTvec(fc.R, normals + 3 * g, nf);
      orc_direct_forcing(ub, uf, nf, s->rho_phys, areas[g], dx, dt, s->wall, fl);
      matvec(fc.R, fl, force_world + 3 * g);
    }
    /* serial spread in ascending marker order, session.hpp:129-144 */
    const double f2l = dt * dt / (s->rho_phys * dx * dx * dx * dx);
    double tf[3] = {0, 0, 0}, tb[3] = {0, 0, 0}, power = 0.0;
    for (long long g = m0; g < m1; ++g) {
      if (!valid[g]) continue;
      const double* fw = force_world + 3 * g;
      double ff[3], xw[3], xf[3], xl[3], fs_[3];
      matTvec(fc.R, fw, ff);
      for (int k = 0; k < 3; ++k) xw[k] = points[3 * g + k] - s->fs.p[k];
      matTvec(fc.R, xw, xf);
      for (int k = 0; k < 3; ++k) xl[k] = xf[k] / dx + half_d[k];
      for (int k = 0; k < 3; ++k) fs_[k] = ff[k] * f2l;
      orc_spread(s->kernel, d, s->F, xl, fs_);
      for (int k = 0; k < 3; ++k) {
        tf[k] = tf[k] + fw[k];
        tb[k] = tb[k] - fw[k];
      }
      const double nfw[3] = {-fw[0], -fw[1], -fw[2]};
      power += dot3(nfw, velocities + 3 * g);
    }
    if (stats) {
      for (int k = 0; k < 3; ++k) {
        stats[7 * b + k] = tf[k];
        stats[7 * b + 3 + k] = tb[k];
      }
      stats[7 * b + 6] = power;
    }
  }

  if (s->frame_mode != 0) { /* session.hpp:148-163 */
    const double acc = dt * dt / dx;
    const double v2p = dx / dt;
#pragma omp parallel for schedule(static)
    for (int k = 0; k < d[2]; ++k)
      for (int j = 0; j < d[1]; ++j)
        for (int i = 0; i < d[0]; ++i) {
          const size_t c = cidx(d, i, j, k);
          const double xf[3] = {(i - half_d[0]) * dx, (j - half_d[1]) * dx, (k - half_d[2]) * dx};
          const double uf[3] = {s->u[3 * c] * v2p, s->u[3 * c + 1] * v2p, s->u[3 * c + 2] * v2p};
          double a[3];
          orc_virtual_force(&fc, xf, uf, a);
          const double ra = s->rho[c] * acc;
          for (int q = 0; q < 3; ++q) s->F[3 * c + q] = s->F[3 * c + q] + ra * a[q];
        }
  }

  orc_collide_and_stream(d, s->periodic, s->tau, s->fa, s->fb, s->F, finite, min_f);
  double* t = s->fa;
  s->fa = s->fb;
  s->fb = t;
  return nonpos;
}

void orc_session_recenter(orc_session* s, const int shift[3]) {
  orc_recenter(s->d, s->dx, s->fa, s->fb, shift, &s->fs);
  double* t = s->fa;
  s->fa = s->fb;
  s->fb = t;
}

/* ======================================================= skinned bodies ==
 * TEST INFRASTRUCTURE: restatement of the robot-side marker refresh and
 * force reduction of CoupledSession::step.  Eigen 3.4 coefficient order as
 * in the rest of this file: mat*vec and dot ((a0 b0 + a1 b1) + a2 b2),
 * cross3, normalized() = v / sqrt(|v|^2) when |v|^2 > 0. */
static void sk_mv(const double* R, const double* v, double* r) {
  for (int i = 0; i < 3; ++i) r[i] = (R[3 * i] * v[0] + R[3 * i + 1] * v[1]) + R[3 * i + 2] * v[2];
}
static void sk_mtv(const double* R, const double* v, double* r) {
  for (int i = 0; i < 3; ++i) r[i] = (R[i] * v[0] + R[3 + i] * v[1]) + R[6 + i] * v[2];
}
static void sk_cross(const double* a, const double* b, double* r) {
  r[0] = a[1] * b[2] - a[2] * b[1];
  r[1] = a[2] * b[0] - a[0] * b[2];
  r[2] = a[0] * b[1] - a[1] * b[0];
}
static double sk_dot(const double* a, const double* b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

/* BoneTransforms::apply (skinning.hpp:101) */
static void sk_apply(const orc_body_pose* P, int b, const double* x, double* xb) {
  sk_mv(P->bone_R[b], x, xb);
  for (int c = 0; c < 3; ++c) xb[c] = xb[c] + P->bone_t[b][c];
}

void orc_update_samples(const orc_skeleton* sk, const orc_body_pose* P, int m, const double* rest,
                        const double* nrest, const double* weights, double* pts, double* vel,
                        double* nrm) {
  const int L = sk->n_links;
  for (int i = 0; i < m; ++i) {
    const double* w = weights + (size_t)i * L;
    const double* x = rest + 3 * i;
    double out[3] = {0, 0, 0}, vo[3] = {0, 0, 0}, nn[3] = {0, 0, 0};
    /* skin_point (skinning.hpp:105-112) */
    for (int b = 0; b < L; ++b) {
      if (w[b] == 0.0) continue;
      double xb[3];
      sk_apply(P, b, x, xb);
      for (int c = 0; c < 3; ++c) out[c] = out[c] + w[b] * xb[c];
    }
    /* skin_point_velocity (skinning.hpp:116-126) */
    for (int b = 0; b < L; ++b) {
      if (w[b] == 0.0) continue;
      double xb[3], d[3], cr[3];
      sk_apply(P, b, x, xb);
      for (int c = 0; c < 3; ++c) d[c] = xb[c] - P->p_world[b][c];
      sk_cross(P->omega_world[b], d, cr);
      for (int c = 0; c < 3; ++c) vo[c] = vo[c] + w[b] * (P->v_origin_world[b][c] + cr[c]);
    }
    /* normals (sampling.hpp:316-319) */
    for (int b = 0; b < L; ++b) {
      if (w[b] == 0.0) continue;
      double rn[3];
      sk_mv(P->bone_R[b], nrest + 3 * i, rn);
      for (int c = 0; c < 3; ++c) nn[c] = nn[c] + w[b] * rn[c];
    }
    const double z = sk_dot(nn, nn);
    if (z > 0.0) {
      const double s = sqrt(z);
      for (int c = 0; c < 3; ++c) nn[c] = nn[c] / s;
    }
    for (int c = 0; c < 3; ++c) {
      pts[3 * i + c] = out[c];
      vel[3 * i + c] = vo[c];
      nrm[3 * i + c] = nn[c];
    }
  }
}

/* accumulate_point_force (dynamics.hpp:216-233) */
static void sk_point_force(const orc_skeleton* sk, const orc_body_pose* P, int link, const double* p,
                           const double* f, double* tau) {
  if (sk->floating_base) {
    double d[3], cr[3], h[3], g[3];
    for (int c = 0; c < 3; ++c) d[c] = p[c] - P->p_world[0][c];
    sk_cross(d, f, cr);
    sk_mtv(P->R_world[0], cr, h);
    for (int c = 0; c < 3; ++c) tau[c] = tau[c] + h[c];
    sk_mtv(P->R_world[0], f, g);
    for (int c = 0; c < 3; ++c) tau[3 + c] = tau[3 + c] + g[c];
  }
  for (int j = link; j > 0; j = sk->parent[j]) {
    if (sk->dof_index[j] < 0) continue; /* not revolute */
    double aw[3], d[3], cr[3];
    sk_mv(P->R_world[j], sk->axis[j], aw);
    for (int c = 0; c < 3; ++c) d[c] = p[c] - P->p_world[j][c];
    sk_cross(aw, d, cr);
    tau[sk->dof_index[j]] = tau[sk->dof_index[j]] + sk_dot(cr, f);
  }
}

void orc_skin_tau(const orc_skeleton* sk, const orc_body_pose* P, int m, const double* rest,
                  const double* weights, const double* fworld, const int* valid, const double* vel,
                  double* tau, double* stats) {
  const int L = sk->n_links;
  for (int d = 0; d < sk->n_dofs; ++d) tau[d] = 0.0;
  for (int k = 0; k < 7; ++k) stats[k] = 0.0;
  for (int i = 0; i < m; ++i) {
    if (!valid[i]) continue;
    const double* f = fworld + 3 * i;
    const double fneg[3] = {-f[0], -f[1], -f[2]};
    const double* w = weights + (size_t)i * L;
    /* accumulate_skinned_force (skinning.hpp:147-156), called with -f_world */
    for (int b = 0; b < L; ++b) {
      if (w[b] == 0.0) continue;
      double p[3], fv[3];
      sk_apply(P, b, rest + 3 * i, p);
      for (int c = 0; c < 3; ++c) fv[c] = w[b] * fneg[c];
      sk_point_force(sk, P, b, p, fv, tau);
    }
    /* CouplingStats (session.hpp:141-143) */
    for (int c = 0; c < 3; ++c) {
      stats[c] = stats[c] + f[c];
      stats[3 + c] = stats[3 + c] - f[c];
    }
    stats[6] = stats[6] + sk_dot(fneg, vel + 3 * i);
  }
}

/* surface_force (empirical.hpp:25-30): -k (n.v) n A on advancing patches */
static void orc_surface_force(const double* n, const double* v, double area, double k, double* f) {
  const double vn = sk_dot(n, v);
  if (vn <= 0.0) {
    f[0] = f[1] = f[2] = 0.0;
    return;
  }
  const double s = ((-k) * vn) * area;
  for (int c = 0; c < 3; ++c) f[c] = s * n[c];
}

void orc_empirical_step(const orc_skeleton* sk, const orc_body_pose* P, int m, const double* rest,
                        const double* nrest, const double* weights, const double* areas, double k,
                        double* tau, double* stats) {
  const int L = sk->n_links;
  double* pts = (double*)malloc(sizeof(double) * 3 * (size_t)(m > 0 ? m : 1));
  double* vel = (double*)malloc(sizeof(double) * 3 * (size_t)(m > 0 ? m : 1));
  double* nrm = (double*)malloc(sizeof(double) * 3 * (size_t)(m > 0 ? m : 1));
  orc_update_samples(sk, P, m, rest, nrest, weights, pts, vel, nrm);
  for (int d = 0; d < sk->n_dofs; ++d) tau[d] = 0.0;
  for (int q = 0; q < 7; ++q) stats[q] = 0.0;
  for (int i = 0; i < m; ++i) {
    double f[3];
    orc_surface_force(nrm + 3 * i, vel + 3 * i, areas[i], k, f);
    if (fabs(f[0]) <= 1e-12 && fabs(f[1]) <= 1e-12 && fabs(f[2]) <= 1e-12) continue; /* isZero */
    const double* w = weights + (size_t)i * L;
    for (int b = 0; b < L; ++b) { /* accumulate_skinned_force(..., f, tau) */
      if (w[b] == 0.0) continue;
      double p[3], fv[3];
      sk_apply(P, b, rest + 3 * i, p);
      for (int c = 0; c < 3; ++c) fv[c] = w[b] * f[c];
      sk_point_force(sk, P, b, p, fv, tau);
    }
    for (int c = 0; c < 3; ++c) stats[3 + c] = stats[3 + c] + f[c];
    stats[6] = stats[6] + sk_dot(f, vel + 3 * i);
  }
  free(pts);
  free(vel);
  free(nrm);
}
