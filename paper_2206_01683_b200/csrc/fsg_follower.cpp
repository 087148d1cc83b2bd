// fsg_follower.cpp -- frame::FrameFollower (frame.hpp:70-125) on the host.
//
// The second-order critically damped tracker that produces the local
// frame's state (p, pd, pdd, q, omega, alpha) from the robot base pose every
// step; its output is the input of fsg_set_frame.  Host scalar code, fp64,
// with Eigen 3.4's coefficient order for the small vector/quaternion algebra
// (the same order as the oracle's stand-in), so the state is bit-identical to
// the reference's (tests/test_follower.py).  Built with -ffp-contract=off.
#include <cmath>
#include <new>

#include "../../include/fsg.h"

struct fsg_follower {
  int mode = FSG_FRAME_TRANSLATION;
  double wn = 5.0;  // 1 / time constant (0.2 s)
  fsg_frame_state f{};
};

namespace {

// Vec3 helpers (Eigen: dot/squaredNorm ((a0*b0 + a1*b1) + a2*b2))
double norm3(const double v[3]) { return std::sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]); }

// Quaternion (w, x, y, z); Eigen's normalize: coefficient order (x,y,z,w),
// squaredNorm reduced as (x*x + z*z) + (y*y + w*w)
void qnormalize(double q[4]) {
  const double n = std::sqrt((q[1] * q[1] + q[3] * q[3]) + (q[2] * q[2] + q[0] * q[0]));
  q[1] = q[1] / n;
  q[2] = q[2] / n;
  q[3] = q[3] / n;
  q[0] = q[0] / n;
}
void qmul(const double a[4], const double b[4], double r[4]) {  // Hamilton product
  const double w = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
  const double x = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
  const double y = a[0] * b[2] + a[2] * b[0] + a[3] * b[1] - a[1] * b[3];
  const double z = a[0] * b[3] + a[3] * b[0] + a[1] * b[2] - a[2] * b[1];
  r[0] = w;
  r[1] = x;
  r[2] = y;
  r[3] = z;
}
// Quaternion(AngleAxis(angle, axis))
void q_from_aa(double angle, const double axis[3], double q[4]) {
  const double ha = 0.5 * angle;
  const double s = std::sin(ha);
  q[0] = std::cos(ha);
  q[1] = s * axis[0];
  q[2] = s * axis[1];
  q[3] = s * axis[2];
}
// quat_exp (types.hpp:71-79): rotation vector -> quaternion, safe near 0
void quat_exp(const double w[3], double q[4]) {
  const double angle = norm3(w);
  if (angle < 1e-12) {
    q[0] = 1.0;
    q[1] = 0.5 * w[0];
    q[2] = 0.5 * w[1];
    q[3] = 0.5 * w[2];
    qnormalize(q);
    return;
  }
  const double axis[3] = {w[0] / angle, w[1] / angle, w[2] / angle};
  q_from_aa(angle, axis, q);
}
// yaw of matrix_to_euler_zyx(q.toRotationMatrix()) (types.hpp:57-68)
double yaw_of(const double q[4]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  const double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
  const double twy = ty * w, twz = tz * w;
  const double txy = ty * x, txz = tz * x;
  const double tyy = ty * y, tzz = tz * z;
  const double r00 = 1.0 - (tyy + tzz), r10 = txy + twz, r20 = txz - twy;
  if (std::abs(r20) < 1.0 - 1e-12) return std::atan2(r10, r00);
  return 0.0;
}
double wrap_angle(double a) {  // types.hpp:81-85
  while (a > M_PI) a -= 2.0 * M_PI;
  while (a < -M_PI) a += 2.0 * M_PI;
  return a;
}

}  // namespace

extern "C" {

int fsg_follower_create(int mode, double time_constant, fsg_follower** out) {
  if (!out) return FSG_EINPUT;
  *out = nullptr;
  if (mode < FSG_FRAME_NONE || mode > FSG_FRAME_FULL || !(time_constant > 0.0)) return FSG_EINPUT;
  fsg_follower* f = new (std::nothrow) fsg_follower();
  if (!f) return FSG_ECUDA;
  f->mode = mode;
  f->wn = 1.0 / time_constant;
  f->f.q[0] = 1.0;
  *out = f;
  return FSG_OK;
}

int fsg_follower_destroy(fsg_follower* f) {
  delete f;
  return FSG_OK;
}

int fsg_follower_reset(fsg_follower* f, const double p[3], double yaw) {
  if (!f || !p) return FSG_EINPUT;
  f->f = fsg_frame_state{};
  f->f.q[0] = 1.0;
  for (int k = 0; k < 3; ++k) f->f.p[k] = p[k];
  if (f->mode == FSG_FRAME_TRANSLATION_YAW || f->mode == FSG_FRAME_FULL) {
    const double w[3] = {0.0, 0.0, yaw};
    quat_exp(w, f->f.q);
  }
  return FSG_OK;
}

int fsg_follower_step(fsg_follower* f, const double tp[3], const double tq[4], double dt) {
  if (!f || !tp || !tq) return FSG_EINPUT;
  fsg_frame_state& s = f->f;
  const double wn = f->wn;
  if (f->mode == FSG_FRAME_NONE) return FSG_OK;
  // frame.hpp:93-95
  for (int k = 0; k < 3; ++k) s.pdd[k] = wn * wn * (tp[k] - s.p[k]) - 2.0 * wn * s.pd[k];
  for (int k = 0; k < 3; ++k) s.pd[k] += dt * s.pdd[k];
  for (int k = 0; k < 3; ++k) s.p[k] += dt * s.pd[k];
  if (f->mode == FSG_FRAME_TRANSLATION) return FSG_OK;
  double err[3];
  if (f->mode == FSG_FRAME_TRANSLATION_YAW) {  // frame.hpp:98-101
    err[0] = 0.0;
    err[1] = 0.0;
    err[2] = wrap_angle(yaw_of(tq) - yaw_of(s.q));
  } else {  // frame.hpp:102-107: AngleAxis of (target * conj(rot)).normalized()
    const double conj[4] = {s.q[0], -s.q[1], -s.q[2], -s.q[3]};
    double dq[4];
    qmul(tq, conj, dq);
    qnormalize(dq);
    const double v[3] = {dq[1], dq[2], dq[3]};
    const double n = norm3(v);
    double angle = 0.0, axis[3] = {1.0, 0.0, 0.0};
    if (n != 0.0) {
      angle = 2.0 * std::atan2(n, std::abs(dq[0]));
      const double sg = dq[0] < 0.0 ? -1.0 : 1.0;
      for (int k = 0; k < 3; ++k) axis[k] = sg < 0.0 ? -v[k] / n : v[k] / n;
    }
    if (angle > M_PI) angle -= 2.0 * M_PI;
    for (int k = 0; k < 3; ++k) err[k] = angle * axis[k];
  }
  // frame.hpp:108-111
  for (int k = 0; k < 3; ++k) s.alpha[k] = wn * wn * err[k] - 2.0 * wn * s.omega[k];
  for (int k = 0; k < 3; ++k) s.omega[k] += dt * s.alpha[k];
  const double wdt[3] = {s.omega[0] * dt, s.omega[1] * dt, s.omega[2] * dt};
  double e[4], r[4];
  quat_exp(wdt, e);
  qmul(e, s.q, r);
  qnormalize(r);
  for (int k = 0; k < 4; ++k) s.q[k] = r[k];
  if (f->mode == FSG_FRAME_TRANSLATION_YAW) {  // frame.hpp:112-118: pin to pure yaw
    const double w[3] = {0.0, 0.0, yaw_of(s.q)};
    quat_exp(w, s.q);
    s.omega[0] = s.omega[1] = 0.0;
    s.alpha[0] = s.alpha[1] = 0.0;
  }
  return FSG_OK;
}

int fsg_follower_state(const fsg_follower* f, fsg_frame_state* out) {
  if (!f || !out) return FSG_EINPUT;
  *out = f->f;
  return FSG_OK;
}

int fsg_follower_set_state(fsg_follower* f, const fsg_frame_state* in) {
  if (!f || !in) return FSG_EINPUT;
  f->f = *in;
  return FSG_OK;
}

int fsg_follower_center(fsg_follower* f, const double base_p[3], const double base_q[4]) {
  if (!f || !base_p || !base_q) return FSG_EINPUT;
  // CoupledSession::center_frame_on_robot (session.hpp:210-221)
  if (f->mode == FSG_FRAME_NONE) {
    const double z[3] = {0.0, 0.0, 0.0};
    return fsg_follower_reset(f, z, 0.0);
  }
  return fsg_follower_reset(f, base_p, f->mode == FSG_FRAME_TRANSLATION ? 0.0 : yaw_of(base_q));
}

}  // extern "C"
