// fishgym_b200/session.hpp -- header-only C++ host over the C ABI (fsg.h).
//
// Mirrors the reference's hot-path API so that FishGym's sim::CoupledSession
// (session.hpp:29-224) can delegate its fluid half to the B200 path:
//
//   reference (fishsim)                         here (fishgym_b200)
//   --------------------------------------------------------------------------
//   UnitMap::validate, LatticeGrid(dims,...)     FluidSession(Config)      (throws InputError)
//   LatticeGrid::reset_to_rest / initialize      reset_to_rest / initialize
//   grid.front() (post-stream f)                 get_f / set_f
//   lbm::collide_and_stream(grid, force)         collide_and_stream (after set_force)
//   lbm::macroscopic(grid, force)                macroscopic
//   lbm::total_mass / total_momentum             total_mass / total_momentum
//   frame::recenter(grid, frame, shift)          recenter
//   frame::FrameFollower(mode, tc) reset/step    FrameFollower reset / step / state
//   CoupledSession::step() fluid half            set_frame + set_markers + step
//   (session.hpp:94-166)                          + marker_forces / stats
//
// Errors follow the reference: invalid configuration throws InputError
// (types.hpp:27-30); CUDA failures throw std::runtime_error; instability is
// reported in StepStatus, never thrown (solver.hpp:13-20).
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../fsg.h"

namespace fishgym_b200 {

class InputError : public std::runtime_error {
 public:
  explicit InputError(const std::string& w) : std::runtime_error(w) {}
};

inline void check(int rc) {
  if (rc == FSG_OK) return;
  const std::string msg = fsg_last_error();
  if (rc == FSG_EINPUT) throw InputError(msg);
  throw std::runtime_error("fsg: " + msg);
}

inline void check_dyn(int rc) {
  if (rc == FSG_OK) return;
  const std::string msg = fsg_dyn_last_error();
  if (rc == FSG_EINPUT) throw InputError(msg);
  throw std::runtime_error("fsg_dyn: " + msg);
}

/// StepStatus (solver.hpp:13-20) + StepOutcome (backend.hpp:37-40).
struct StepStatus {
  bool finite = true;
  double min_f = 0.0;
  int n_nonpositive_rho = 0;
  int out_of_bounds_markers = 0;
  bool stable(double negative_tolerance = 1e-3) const {
    return finite && min_f > -negative_tolerance && n_nonpositive_rho == 0;
  }
};

/// FrameState (frame.hpp:13-20), world frame; q = (w, x, y, z).
struct FrameState {
  std::array<double, 3> p{}, pd{}, pdd{}, omega{}, alpha{};
  std::array<double, 4> q{1.0, 0.0, 0.0, 0.0};
};

struct Config : fsg_config {
  Config() { fsg_config_default(this); }
};

/// frame::FrameFollower (frame.hpp:70-125): the critically damped tracker of
/// the robot base; state() is what FluidSession::set_frame takes.
class FrameFollower {
 public:
  explicit FrameFollower(int mode = FSG_FRAME_TRANSLATION, double time_constant = 0.2) {
    check(fsg_follower_create(mode, time_constant, &h_));
  }
  ~FrameFollower() { fsg_follower_destroy(h_); }
  FrameFollower(const FrameFollower&) = delete;
  FrameFollower& operator=(const FrameFollower&) = delete;

  void reset(const std::array<double, 3>& p, double yaw) { check(fsg_follower_reset(h_, p.data(), yaw)); }
  void step(const std::array<double, 3>& target_p, const std::array<double, 4>& target_q, double dt) {
    check(fsg_follower_step(h_, target_p.data(), target_q.data(), dt));
  }
  FrameState state() const {
    fsg_frame_state c{};
    check(fsg_follower_state(h_, &c));
    FrameState f;
    for (int k = 0; k < 3; ++k) {
      f.p[k] = c.p[k];
      f.pd[k] = c.pd[k];
      f.pdd[k] = c.pdd[k];
      f.omega[k] = c.omega[k];
      f.alpha[k] = c.alpha[k];
    }
    for (int k = 0; k < 4; ++k) f.q[k] = c.q[k];
    return f;
  }

 private:
  fsg_follower* h_ = nullptr;
};

class FluidSession {
 public:
  explicit FluidSession(const Config& cfg) : dims_{cfg.dims[0], cfg.dims[1], cfg.dims[2]} {
    check(fsg_create(&cfg, &h_));
    n_ = static_cast<size_t>(dims_[0]) * dims_[1] * dims_[2];
  }
  ~FluidSession() { fsg_destroy(h_); }
  FluidSession(const FluidSession&) = delete;
  FluidSession& operator=(const FluidSession&) = delete;

  size_t n_cells() const { return n_; }
  std::array<int, 3> dims() const { return dims_; }

  // ---- LatticeGrid ----------------------------------------------------------
  void reset_to_rest() { check(fsg_reset_rest(h_)); }
  void initialize(const std::vector<double>& rho, const std::vector<double>& u) {
    check(fsg_initialize(h_, rho.data(), u.data()));
  }
  void set_f(const std::vector<double>& f) { check(fsg_set_f(h_, f.data())); }
  std::vector<double> get_f() const {
    std::vector<double> f(19 * n_);
    check(fsg_get_f(h_, f.data()));
    return f;
  }

  // ---- lbm::solver ------------------------------------------------------------
  void set_force(const std::vector<double>* F) { check(fsg_set_force(h_, F ? F->data() : nullptr)); }
  StepStatus collide_and_stream() { return status_of(call_status(fsg_collide_and_stream)); }
  int macroscopic(std::vector<double>& rho, std::vector<double>& u) {
    rho.resize(n_);
    u.resize(3 * n_);
    int nonpos = 0;
    check(fsg_macroscopic(h_, rho.data(), u.data(), &nonpos));
    return nonpos;
  }
  double total_mass() const {
    double m = 0.0;
    check(fsg_total_mass(h_, &m));
    return m;
  }
  std::array<double, 3> total_momentum() const {
    std::array<double, 3> p{};
    check(fsg_total_momentum(h_, p.data()));
    return p;
  }

  // ---- frame ------------------------------------------------------------------
  void set_frame(const FrameState& f) {
    fsg_frame_state c{};
    for (int k = 0; k < 3; ++k) {
      c.p[k] = f.p[k];
      c.pd[k] = f.pd[k];
      c.pdd[k] = f.pdd[k];
      c.omega[k] = f.omega[k];
      c.alpha[k] = f.alpha[k];
    }
    for (int k = 0; k < 4; ++k) c.q[k] = f.q[k];
    check(fsg_set_frame(h_, &c));
  }
  std::array<double, 3> frame_origin() const {
    fsg_frame_state c{};
    check(fsg_get_frame(h_, &c));
    return {c.p[0], c.p[1], c.p[2]};
  }
  void recenter(const std::array<int, 3>& shift) { check(fsg_recenter(h_, shift.data())); }

  // ---- coupled step (session.hpp:94-166) ------------------------------------
  /// World-frame marker state of all bodies (what robot::update_samples
  /// produces); body b owns markers [offsets[b], offsets[b+1]).
  void set_markers(const std::vector<int64_t>& offsets, const std::vector<double>& points,
                   const std::vector<double>& velocities, const std::vector<double>& normals,
                   const std::vector<double>& areas) {
    m_ = offsets.empty() ? 0 : static_cast<size_t>(offsets.back());
    nb_ = offsets.empty() ? 0 : static_cast<int>(offsets.size()) - 1;
    check(fsg_set_markers(h_, nb_, offsets.data(), points.data(), velocities.data(),
                          normals.data(), areas.data()));
  }
  StepStatus step() { return status_of(call_status(fsg_step)); }
  /// Per-marker world force on the FLUID (N) and CouplingStats per body
  /// (force on fluid[3], force on body[3], power on body).
  void marker_forces(std::vector<double>& force_world, std::vector<int>& valid,
                     std::vector<double>& stats) const {
    force_world.resize(3 * m_);
    valid.resize(m_);
    stats.resize(7 * static_cast<size_t>(nb_ > 0 ? nb_ : 1));
    check(fsg_get_marker_forces(h_, force_world.data(), valid.data(), stats.data()));
  }

  // ---- skinned bodies on the device ---------------------
  /// Register the robots' SurfaceSamples (sampling.hpp): rest points/normals
  /// (base at identity), blend weights (n_links(b) per marker, concatenated
  /// over bodies), areas, and each robot's topology.  From then on every
  /// step() skins the markers on the device (update_samples,
  /// sampling.hpp:307-322) from the pose given to set_pose().
  void set_skin(const std::vector<int64_t>& offsets, const std::vector<fsg_skeleton>& skeletons,
                const std::vector<double>& rest_points, const std::vector<double>& rest_normals,
                const std::vector<double>& weights, const std::vector<double>& areas) {
    m_ = offsets.empty() ? 0 : static_cast<size_t>(offsets.back());
    nb_ = offsets.empty() ? 0 : static_cast<int>(offsets.size()) - 1;
    check(fsg_set_skin(h_, nb_, offsets.data(), skeletons.data(), rest_points.data(),
                       rest_normals.data(), weights.data(), areas.data()));
    nt_ = 0;
    for (const auto& k : skeletons) nt_ += static_cast<size_t>(k.n_dofs);
  }
  /// This step's pose of every robot: BoneTransforms::of (skinning.hpp:85-102)
  /// and the KinematicsCache fields of forward_kinematics (dynamics.hpp:23-61).
  void set_pose(const std::vector<fsg_body_pose>& poses) { check(fsg_set_pose(h_, poses.data())); }
  /// tau_ext of every robot (concatenated; session.hpp:139-140) and the
  /// CouplingStats (7 per body) of the last step.
  void body_wrench(std::vector<double>& tau_ext, std::vector<double>& stats) const {
    tau_ext.resize(nt_);
    stats.resize(7 * static_cast<size_t>(nb_ > 0 ? nb_ : 1));
    check(fsg_get_body_wrench(h_, tau_ext.data(), stats.data()));
  }

  fsg_session* handle() const { return h_; }

 private:
  template <class Fn>
  fsg_status call_status(Fn fn) {
    fsg_status st{};
    check(fn(h_, &st));
    return st;
  }
  static StepStatus status_of(const fsg_status& s) {
    StepStatus r;
    r.finite = s.finite != 0;
    r.min_f = s.min_f;
    r.n_nonpositive_rho = s.n_nonpositive_rho;
    r.out_of_bounds_markers = s.out_of_bounds_markers;
    return r;
  }

  fsg_session* h_ = nullptr;
  std::array<int, 3> dims_{};
  size_t n_ = 0;
  size_t m_ = 0;
  size_t nt_ = 0;
  int nb_ = 0;
};

/// A batch of robots of one skeleton on the device:
/// robot::integrate / buoyancy_gravity_forces (dynamics.hpp:237-289) for
/// every robot per call.  fsg_robot mirrors robot::Skeleton + Bladder
/// (skeleton.hpp:16-93); an invalid skeleton throws InputError with
/// Skeleton::validate's message.
class RobotDynamics {
 public:
  RobotDynamics(const fsg_robot& robot, int n_envs, int device = 0) : n_envs_(n_envs) {
    check_dyn(fsg_dyn_create(&robot, n_envs, device, &h_));
    nd_ = fsg_dyn_n_dofs(h_);
    nj_ = fsg_dyn_n_joints(h_);
  }
  ~RobotDynamics() { fsg_dyn_destroy(h_); }
  RobotDynamics(const RobotDynamics&) = delete;
  RobotDynamics& operator=(const RobotDynamics&) = delete;

  int n_dofs() const { return nd_; }
  int n_joints() const { return nj_; }
  void set_states(const std::vector<fsg_joint_state>& st) { check_dyn(fsg_dyn_set_state(h_, st.data())); }
  std::vector<fsg_joint_state> states() {
    std::vector<fsg_joint_state> st(n_envs_);
    check_dyn(fsg_dyn_get_state(h_, st.data()));
    return st;
  }
  /// session.hpp:169-175 for every robot: actuation [n_envs * n_joints],
  /// tau_ext [n_envs * n_dofs] (empty: zero); g_hydro / gravity nullable.
  /// Returns the FSG_DYN_* flags per robot.
  std::vector<int> step(const std::vector<double>& actuation, const std::vector<double>& tau_ext,
                        double rho_fluid, const double* g_hydro, double dt, int substeps,
                        const double* gravity) {
    std::vector<int> flags(n_envs_);
    check_dyn(fsg_dyn_step(h_, actuation.data(), tau_ext.empty() ? nullptr : tau_ext.data(), rho_fluid,
                           g_hydro, dt, substeps, gravity, flags.data()));
    return flags;
  }
  fsg_dyn* handle() { return h_; }

 private:
  fsg_dyn* h_ = nullptr;
  int n_envs_ = 0, nd_ = 0, nj_ = 0;
};

}  // namespace fishgym_b200
