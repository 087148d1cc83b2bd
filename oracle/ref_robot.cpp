// oracle/_ref robot side -- TEST INFRASTRUCTURE ONLY.
//
// Compiles the REFERENCE's robot, empirical and session headers, unmodified,
// straight from /root/reference/proj/include (robot/{spatial,skeleton,
// dynamics,skinning,sampling,meshes,model_builder,gait}, empirical/empirical,
// sim/{backend,session}) against the Eigen stand-in in oracle/eigen_shim,
// and exposes them through a flat extern "C" surface so that the tests can
// pin the device robot path (skinning + tau_ext, articulated dynamics,
// empirical drag, the whole CoupledSession::step with its follower and
// recentre trigger) and the C restatements to the reference's own code.
// Nothing here restates reference arithmetic: every function below calls the
// reference's.
//
// Packed layouts (doubles):
//   link   [40]: parent, joint (0 Free, 1 Revolute, 2 Fixed), joint_origin[3],
//                joint_rotation[9] (row-major), axis[3], mass, com[3],
//                inertia_com[9] (row-major), stiffness, damping, q_rest,
//                limit_lo, limit_hi, torque_limit, displaced_volume,
//                volume_centroid[3]
//   bladder [8]: volume, volume_min, volume_max, rate_bound, centroid[3], 0
//   state      : base_pos[3], base_quat[4] (w, x, y, z), q[n_joints], v[n_dofs]
//   stats   [8]: force_on_fluid[3], force_on_body[3], power_on_body, oob
//
// Built by oracle/Makefile into oracle/_ref/libfishref.so; never shipped.

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "fishsim/empirical/empirical.hpp"
#include "fishsim/robot/dynamics.hpp"
#include "fishsim/robot/model_builder.hpp"
#include "fishsim/robot/sampling.hpp"
#include "fishsim/robot/skinning.hpp"
#include "fishsim/sim/session.hpp"

using namespace fishsim;
using robot::JointState;
using robot::RobotModel;
using robot::Skeleton;

namespace {

thread_local char g_rerr[512];

Vec3 v3(const double* p) { return Vec3(p[0], p[1], p[2]); }
void put3(double* p, const Vec3& v) {
  p[0] = v.x();
  p[1] = v.y();
  p[2] = v.z();
}
void put33(double* p, const Mat3& m) {  // row-major
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) p[3 * i + j] = m(i, j);
}
Mat3 get33(const double* p) {
  Mat3 m;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m(i, j) = p[3 * i + j];
  return m;
}

void put_state(const Skeleton& sk, const JointState& st, double* out) {
  put3(out, st.base_pos);
  out[3] = st.base_quat.w();
  out[4] = st.base_quat.x();
  out[5] = st.base_quat.y();
  out[6] = st.base_quat.z();
  for (int j = 0; j < sk.n_joints(); ++j) out[7 + j] = st.q[j];
  for (int d = 0; d < sk.n_dofs(); ++d) out[7 + sk.n_joints() + d] = st.v[d];
}
JointState get_state(const Skeleton& sk, const double* in) {
  JointState st = JointState::zero(sk);
  st.base_pos = v3(in);
  st.base_quat = Quat(in[3], in[4], in[5], in[6]);
  for (int j = 0; j < sk.n_joints(); ++j) st.q[j] = in[7 + j];
  for (int d = 0; d < sk.n_dofs(); ++d) st.v[d] = in[7 + sk.n_joints() + d];
  return st;
}
VecX get_vec(const double* p, int n) {
  VecX v = VecX::Zero(n);
  if (p)
    for (int k = 0; k < n; ++k) v[k] = p[k];
  return v;
}
void put_stats(const ib::CouplingStats& s, double* out) {
  put3(out, s.total_force_on_fluid);
  put3(out + 3, s.total_force_on_body);
  out[6] = s.power_on_body;
  out[7] = s.out_of_bounds_markers;
}

struct Model {
  RobotModel m;
};
struct Samples {
  robot::SurfaceSamples s;
};

template <class F>
int guarded(F f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    std::snprintf(g_rerr, sizeof g_rerr, "%s", e.what());
    return 1;
  }
}

}  // namespace

extern "C" {

const char* ref_robot_last_error() { return g_rerr; }

// ---------------------------------------------------------------- models ---
/// build_fish_model(koi_design() / eel_design() / flatfish_design())
/// (model_builder.hpp:104-264)
void* ref_model_build(const char* design) {
  Model* h = nullptr;
  guarded([&] {
    const std::string d(design);
    robot::FishDesign fd = d == "eel"        ? robot::eel_design()
                           : d == "flatfish" ? robot::flatfish_design()
                           : d == "koi"      ? robot::koi_design()
                                             : throw InputError("unknown design " + d);
    auto m = std::make_unique<Model>();
    m->m = robot::build_fish_model(fd);
    h = m.release();
  });
  return h;
}
void ref_model_destroy(void* h) { delete static_cast<Model*>(h); }
/// {n_links, n_joints, n_dofs, floating_base, n_vertices, n_triangles}
void ref_model_info(void* h, int* out) {
  const auto& m = static_cast<Model*>(h)->m;
  out[0] = m.skeleton.n_links();
  out[1] = m.skeleton.n_joints();
  out[2] = m.skeleton.n_dofs();
  out[3] = m.skeleton.floating_base();
  out[4] = static_cast<int>(m.mesh.vertices.size());
  out[5] = static_cast<int>(m.mesh.triangles.size());
}
void ref_model_links(void* h, double* out) {
  const auto& sk = static_cast<Model*>(h)->m.skeleton;
  for (int i = 0; i < sk.n_links(); ++i) {
    const auto& l = sk.links[i];
    double* o = out + 40 * i;
    o[0] = l.parent;
    o[1] = l.joint == robot::JointType::Free ? 0 : l.joint == robot::JointType::Revolute ? 1 : 2;
    put3(o + 2, l.joint_origin);
    put33(o + 5, l.joint_rotation);
    put3(o + 14, l.axis);
    o[17] = l.mass;
    put3(o + 18, l.com);
    put33(o + 21, l.inertia_com);
    o[30] = l.stiffness;
    o[31] = l.damping;
    o[32] = l.q_rest;
    o[33] = l.limit_lo;
    o[34] = l.limit_hi;
    o[35] = l.torque_limit;
    o[36] = l.displaced_volume;
    put3(o + 37, l.volume_centroid);
  }
}
void ref_model_bladder(void* h, double* out) {
  const auto& b = static_cast<Model*>(h)->m.skeleton.bladder;
  out[0] = b.volume;
  out[1] = b.volume_min;
  out[2] = b.volume_max;
  out[3] = b.rate_bound;
  put3(out + 4, b.centroid);
  out[7] = 0.0;
}
/// mesh vertices [3 nv], triangles [3 nt], weights [nv][n_links]
void ref_model_mesh(void* h, double* verts, int* tris, double* weights) {
  const auto& m = static_cast<Model*>(h)->m;
  for (size_t v = 0; v < m.mesh.vertices.size(); ++v) put3(verts + 3 * v, m.mesh.vertices[v]);
  for (size_t t = 0; t < m.mesh.triangles.size(); ++t)
    for (int k = 0; k < 3; ++k) tris[3 * t + k] = m.mesh.triangles[t][k];
  const int nl = m.skeleton.n_links();
  for (size_t v = 0; v < m.mesh.vertices.size(); ++v)
    for (int b = 0; b < nl; ++b) weights[nl * v + b] = m.mesh.weights(v, b);
}
/// Skeleton::validate (skeleton.hpp:96-120) of a packed skeleton; returns 0
/// or 1 with the InputError message in ref_robot_last_error().
int ref_skeleton_validate(int n_links, const double* links) {
  return guarded([&] {
    Skeleton sk;
    for (int i = 0; i < n_links; ++i) {
      const double* o = links + 40 * i;
      robot::Link l;
      l.name = "l" + std::to_string(i);
      l.parent = static_cast<int>(o[0]);
      l.joint = o[1] == 0 ? robot::JointType::Free
                : o[1] == 1 ? robot::JointType::Revolute
                            : robot::JointType::Fixed;
      l.joint_origin = v3(o + 2);
      l.joint_rotation = get33(o + 5);
      l.axis = v3(o + 14);
      l.mass = o[17];
      l.com = v3(o + 18);
      l.inertia_com = get33(o + 21);
      sk.links.push_back(l);
    }
    sk.validate();
  });
}

// --------------------------------------------------------------- samples ---
/// sample_surface(mesh, spacing, seed) (sampling.hpp:164-303)
void* ref_samples_create(void* model, double spacing, uint64_t seed) {
  Samples* h = nullptr;
  guarded([&] {
    auto s = std::make_unique<Samples>();
    s->s = robot::sample_surface(static_cast<Model*>(model)->m.mesh, spacing, seed);
    h = s.release();
  });
  return h;
}
void ref_samples_destroy(void* h) { delete static_cast<Samples*>(h); }
int64_t ref_samples_n(void* h) { return static_cast<int64_t>(static_cast<Samples*>(h)->s.size()); }
/// rest points/normals [3n], areas [n], weights [n][n_links]
void ref_samples_get(void* h, double* rest_points, double* rest_normals, double* areas,
                     double* weights) {
  const auto& s = static_cast<Samples*>(h)->s;
  const int nl = static_cast<int>(s.weights.cols());
  for (size_t i = 0; i < s.size(); ++i) {
    put3(rest_points + 3 * i, s.rest_points[i]);
    put3(rest_normals + 3 * i, s.rest_normals[i]);
    areas[i] = s.areas[i];
    for (int b = 0; b < nl; ++b) weights[nl * i + b] = s.weights(i, b);
  }
}

// -------------------------------------------------------------- dynamics ---
/// forward_kinematics (dynamics.hpp:23-62) + BoneTransforms::of
/// (skinning.hpp:85-102) + RestPose::of: per link R_world[9], p_world[3],
/// v_origin_world[3], omega_world[3], bone_R[9], bone_t[3] = 30 doubles
void ref_kinematics(void* model, const double* state, double* out) {
  const auto& sk = static_cast<Model*>(model)->m.skeleton;
  const JointState st = get_state(sk, state);
  const auto kc = robot::forward_kinematics(sk, st);
  const auto rest = robot::RestPose::of(sk);
  const auto bt = robot::BoneTransforms::of(kc, rest);
  for (int i = 0; i < sk.n_links(); ++i) {
    double* o = out + 30 * i;
    put33(o, kc.R_world[i]);
    put3(o + 9, kc.p_world[i]);
    put3(o + 12, kc.v_origin_world[i]);
    put3(o + 15, kc.omega_world[i]);
    put33(o + 18, bt.R[i]);
    put3(o + 27, bt.t[i]);
  }
}
/// mass_matrix (dynamics.hpp:66-114), column-major nd x nd
void ref_mass_matrix(void* model, const double* state, double* M) {
  const auto& sk = static_cast<Model*>(model)->m.skeleton;
  const JointState st = get_state(sk, state);
  const MatX m = robot::mass_matrix(sk, robot::forward_kinematics(sk, st));
  std::memcpy(M, m.data(), sizeof(double) * m.size());
}
/// bias_forces (dynamics.hpp:118-154)
void ref_bias_forces(void* model, const double* state, const double* g, double* c) {
  const auto& sk = static_cast<Model*>(model)->m.skeleton;
  const JointState st = get_state(sk, state);
  const VecX v = robot::bias_forces(sk, st, robot::forward_kinematics(sk, st), v3(g));
  std::memcpy(c, v.data(), sizeof(double) * v.size());
}
/// The robot half of CoupledSession::step (session.hpp:167-175): hydro on
/// the pre-step kinematics, then integrate(actuation, tau_ext + hydro, dt,
/// substeps, gravity 0).  bladder_volume < 0: the model's.  Returns 0, or 1
/// on NumericalError (state then holds the substeps done before it).
int ref_robot_step(void* model, double* state, const double* actuation, const double* tau_ext,
                   double rho, const double* g_hydro, double bladder_volume, double dt,
                   int substeps) {
  Skeleton sk = static_cast<Model*>(model)->m.skeleton;
  if (bladder_volume >= 0.0) sk.bladder.volume = bladder_volume;
  JointState st = get_state(sk, state);
  const int rc = guarded([&] {
    const auto kc = robot::forward_kinematics(sk, st);
    const VecX hydro = robot::buoyancy_gravity_forces(sk, kc, sk.bladder, rho, v3(g_hydro));
    robot::integrate(sk, st, get_vec(actuation, sk.n_joints()),
                     get_vec(tau_ext, sk.n_dofs()) + hydro, dt, substeps, Vec3::Zero());
  });
  put_state(sk, st, state);
  return rc;
}
/// update_samples (sampling.hpp:307-322) at `state`: points, velocities,
/// normals [3n] (world)
void ref_update_samples(void* model, void* samples, const double* state, double* points,
                        double* velocities, double* normals) {
  const auto& sk = static_cast<Model*>(model)->m.skeleton;
  auto s = static_cast<Samples*>(samples)->s;
  const JointState st = get_state(sk, state);
  const auto kc = robot::forward_kinematics(sk, st);
  robot::update_samples(sk, kc, robot::RestPose::of(sk), s);
  for (size_t i = 0; i < s.size(); ++i) {
    put3(points + 3 * i, s.points[i]);
    put3(velocities + 3 * i, s.velocities[i]);
    put3(normals + 3 * i, s.normals[i]);
  }
}
/// The tau_ext / CouplingStats loop of CoupledSession::step
/// (session.hpp:127-143) for given per-sample forces on the fluid f_world
/// [3n] and validity [n]: accumulate_skinned_force(-f_world) in ascending
/// sample order.  tau [n_dofs], stats [8]
void ref_skinned_tau(void* model, void* samples, const double* state, const double* f_world,
                     const int* valid, double* tau, double* stats) {
  const auto& sk = static_cast<Model*>(model)->m.skeleton;
  auto s = static_cast<Samples*>(samples)->s;
  const JointState st = get_state(sk, state);
  const auto kc = robot::forward_kinematics(sk, st);
  const auto rest = robot::RestPose::of(sk);
  robot::update_samples(sk, kc, rest, s);
  const auto bt = robot::BoneTransforms::of(kc, rest);
  VecX t = VecX::Zero(sk.n_dofs());
  ib::CouplingStats cs;
  for (size_t i = 0; i < s.size(); ++i) {
    if (!valid[i]) {
      ++cs.out_of_bounds_markers;
      continue;
    }
    const Vec3 f = v3(f_world + 3 * i);
    robot::accumulate_skinned_force(sk, kc, bt, s.weights.row(i), s.rest_points[i], -f, t);
    cs.total_force_on_fluid += f;
    cs.total_force_on_body -= f;
    cs.power_on_body += (-f).dot(s.velocities[i]);
  }
  std::memcpy(tau, t.data(), sizeof(double) * t.size());
  put_stats(cs, stats);
}

// ------------------------------------------------------------- empirical ---
/// empirical::EmpiricalBackend (empirical.hpp:36-110)
void* ref_emp_create(double dt, int substeps, double rho, const double* gravity,
                     double spacing, double k) {
  empirical::EmpiricalBackend* h = nullptr;
  guarded([&] {
    empirical::EmpiricalBackend::Config c;
    c.dt = dt;
    c.substeps = substeps;
    c.rho_fluid = rho;
    c.gravity = v3(gravity);
    c.marker_spacing = spacing;
    c.params.k = k;
    h = new empirical::EmpiricalBackend(c);
  });
  return h;
}
void ref_emp_destroy(void* h) { delete static_cast<empirical::EmpiricalBackend*>(h); }
int ref_emp_add_robot(void* h, void* model, const double* pos, double yaw, uint64_t seed) {
  int r = -1;
  guarded([&] {
    sim::RobotStart st;
    st.position = v3(pos);
    st.yaw = yaw;
    r = static_cast<empirical::EmpiricalBackend*>(h)->add_robot(static_cast<Model*>(model)->m,
                                                                  st, seed);
  });
  return r;
}

// ------------------------------------------------ backends (both kinds) ---
static sim::Backend* backend(void* h, int kind) {
  if (kind == 0) return static_cast<empirical::EmpiricalBackend*>(h);
  return static_cast<sim::CoupledSession*>(h);
}
/// kind: 0 EmpiricalBackend, 1 CoupledSession
void ref_be_set_actuation(void* h, int kind, int i, const double* act) {
  auto* b = backend(h, kind);
  b->set_actuation(i, get_vec(act, b->robot(i).skeleton.n_joints()));
}
void ref_be_change_bladder(void* h, int kind, int i, double dv) {
  backend(h, kind)->change_bladder(i, dv);
}
/// Backend::step: returns {stable, out_of_bounds_markers} packed as stable + 2*oob
int ref_be_step(void* h, int kind, int* oob) {
  int stable = 0;
  const int rc = guarded([&] {
    const auto o = backend(h, kind)->step();
    stable = o.stable;
    if (oob) *oob = o.out_of_bounds_markers;
  });
  return rc ? -1 : stable;
}
/// robot i: state (packed), tau_ext [n_dofs], stats [8], bladder volume
void ref_be_robot(void* h, int kind, int i, double* state, double* tau, double* stats,
                  double* bladder_volume) {
  const auto& r = backend(h, kind)->robot(i);
  if (state) put_state(r.skeleton, r.state, state);
  if (tau) std::memcpy(tau, r.tau_ext.data(), sizeof(double) * r.tau_ext.size());
  if (stats) put_stats(r.stats, stats);
  if (bladder_volume) *bladder_volume = r.skeleton.bladder.volume;
}
void ref_be_set_state(void* h, int kind, int i, const double* state) {
  auto& r = backend(h, kind)->robot(i);
  r.state = get_state(r.skeleton, state);
}
/// robot i's samples as the last step left them: points, velocities, normals [3n]
void ref_be_samples(void* h, int kind, int i, double* points, double* velocities,
                    double* normals) {
  const auto& s = backend(h, kind)->robot(i).samples;
  for (size_t k = 0; k < s.size(); ++k) {
    if (points) put3(points + 3 * k, s.points[k]);
    if (velocities) put3(velocities + 3 * k, s.velocities[k]);
    if (normals) put3(normals + 3 * k, s.normals[k]);
  }
}
int64_t ref_be_n_samples(void* h, int kind, int i) {
  return static_cast<int64_t>(backend(h, kind)->robot(i).samples.size());
}

// ------------------------------------------------------- CoupledSession ---
/// sim::CoupledSession (session.hpp:29-241), unmodified: kernel 0 Peskin4 /
/// 1 Roma3; wall 0 Slip / 1 NoSlip; frame_mode 0 None .. 3 Full.
void* ref_cs_create(int nx, int ny, int nz, double dx, double dt, double rho, double nu,
                    int kernel, int wall, int frame_mode, double frame_tc, double recenter_cells,
                    const double* gravity, int substeps, double marker_spacing, int tracked) {
  sim::CoupledSession* h = nullptr;
  guarded([&] {
    sim::SessionConfig c;
    c.dims = {nx, ny, nz};
    c.units.dx = dx;
    c.units.dt_phys = dt;
    c.units.rho_phys = rho;
    c.units.nu_phys = nu;
    c.kernel.family = kernel == 0 ? ib::IBKernel::Family::Peskin4 : ib::IBKernel::Family::Roma3;
    c.wall = wall == 0 ? ib::WallCondition::Slip : ib::WallCondition::NoSlip;
    c.frame_mode = static_cast<frame::FollowMode>(frame_mode);
    c.frame_time_constant = frame_tc;
    c.recenter_threshold_cells = recenter_cells;
    c.gravity = v3(gravity);
    c.substeps = substeps;
    c.marker_spacing = marker_spacing;
    c.tracked_robot = tracked;
    h = new sim::CoupledSession(c);
  });
  return h;
}
void ref_cs_destroy(void* h) { delete static_cast<sim::CoupledSession*>(h); }
int ref_cs_add_robot(void* h, void* model, const double* pos, double yaw, uint64_t seed) {
  int r = -1;
  guarded([&] {
    sim::RobotStart st;
    st.position = v3(pos);
    st.yaw = yaw;
    r = static_cast<sim::CoupledSession*>(h)->add_robot(static_cast<Model*>(model)->m, st, seed);
  });
  return r;
}
/// frame state: p, pd, pdd, q(w,x,y,z), omega, alpha = 19 doubles
void ref_cs_frame(void* h, double* out) {
  const auto& f = static_cast<sim::CoupledSession*>(h)->frame_state();
  put3(out, f.p);
  put3(out + 3, f.pd);
  put3(out + 6, f.pdd);
  out[9] = f.rot.w();
  out[10] = f.rot.x();
  out[11] = f.rot.y();
  out[12] = f.rot.z();
  put3(out + 13, f.omega);
  put3(out + 16, f.alpha);
}
/// post-stream distributions, direction-major [19 * n]
void ref_cs_get_f(void* h, double* f) {
  const auto& g = static_cast<sim::CoupledSession*>(h)->grid();
  const auto& a = g.front();
  std::memcpy(f, a.data(), sizeof(double) * a.size());
}
/// bare macroscopic fields of the last step
void ref_cs_macro(void* h, double* rho, double* u) {
  const auto& m = static_cast<sim::CoupledSession*>(h)->macro();
  for (size_t c = 0; c < m.rho.size(); ++c) {
    rho[c] = m.rho[c];
    put3(u + 3 * c, m.u[c]);
  }
}

}  // extern "C"
