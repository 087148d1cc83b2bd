// oracle/_ref driver -- TEST INFRASTRUCTURE ONLY.
//
// Compiles the REFERENCE's own hot-path headers, unmodified, straight from
// /root/reference/proj/include (core/{types,units,rng}, lbm/{lattice,solver},
// ib/{kernel,coupling}, frame/frame) against the Eigen stand-in in
// oracle/eigen_shim, and exposes them through a flat extern "C" surface so
// that Python tests can (1) pin the C restatement in oracle/fsg_oracle.c and
// (2) generate golden fixtures under tests/golden/.
//
// The only code here that is not the reference's is the orchestration of the
// fluid half of CoupledSession::step (session.hpp:94-166, restated below
// because session.hpp drags in robot/, which needs dynamic-size Eigen) with
// the robot's marker provider replaced by caller-supplied world-frame marker
// state (points, velocities, normals, areas).  Every arithmetic kernel that
// step calls is the reference's own function.
//
// Built by oracle/Makefile into oracle/_ref/libfishref.so; never shipped as
// product, never linked by paper_2206_01683_b200.

#include <cstdint>
#include <cstring>
#include <memory>
#include <vector>

#include "fishsim/core/rng.hpp"
#include "fishsim/core/types.hpp"
#include "fishsim/core/units.hpp"
#include "fishsim/frame/frame.hpp"
#include "fishsim/ib/coupling.hpp"
#include "fishsim/ib/kernel.hpp"
#include "fishsim/lbm/lattice.hpp"
#include "fishsim/lbm/solver.hpp"
#include "fishsim/lbm/vtk.hpp"
#include "fishsim/core/csv.hpp"

using namespace fishsim;

namespace {

struct RefSession {
  Index3 dims;
  UnitMap units;
  lbm::LatticeGrid grid;
  lbm::BodyForceField force;
  lbm::FluidMacro macro;
  ib::IBKernel kernel;
  ib::WallCondition wall = ib::WallCondition::Slip;
  frame::FollowMode frame_mode = frame::FollowMode::None;
  frame::FrameState fs;
  std::vector<Vec3> sample_force_world;
  std::vector<char> sample_valid;
};

UnitMap make_units(double dx, double dt, double rho, double nu) {
  UnitMap u;
  u.dx = dx;
  u.dt_phys = dt;
  u.rho_phys = rho;
  u.nu_phys = nu;
  return u;
}

Vec3 v3(const double* p) { return Vec3(p[0], p[1], p[2]); }
void put3(double* p, const Vec3& v) {
  p[0] = v.x();
  p[1] = v.y();
  p[2] = v.z();
}

// session.hpp:77-85
Vec3 cell_frame_position(const RefSession& s, int i, int j, int k) {
  return Vec3((i - 0.5 * (s.dims[0] - 1)) * s.units.dx, (j - 0.5 * (s.dims[1] - 1)) * s.units.dx,
              (k - 0.5 * (s.dims[2] - 1)) * s.units.dx);
}
Vec3 frame_to_lattice(const RefSession& s, const Vec3& x_frame) {
  return x_frame / s.units.dx + 0.5 * Vec3(s.dims[0] - 1, s.dims[1] - 1, s.dims[2] - 1);
}

thread_local char g_err[512];

}  // namespace

extern "C" {

// lbm::write_vtk (vtk.hpp:15-38) on caller fields; 0 ok, 1 InputError
int ref_write_vtk(const char* path, int nx, int ny, int nz, const double* rho, const double* u,
                  double dx, double dt, double rho_phys, double nu, const double* origin) {
  try {
    lbm::FluidMacro m;
    m.resize(Index3{nx, ny, nz});
    for (size_t c = 0; c < m.rho.size(); ++c) {
      m.rho[c] = rho[c];
      m.u[c] = Vec3(u[3 * c], u[3 * c + 1], u[3 * c + 2]);
    }
    UnitMap un;
    un.dx = dx;
    un.dt_phys = dt;
    un.rho_phys = rho_phys;
    un.nu_phys = nu;
    lbm::write_vtk(path, m, un, Vec3(origin[0], origin[1], origin[2]));
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

// CsvWriter (csv.hpp:27-66): header + nrows rows of ncols values
int ref_csv_write(const char* path, int ncols, const char* const* names, int nrows,
                  const double* values) {
  try {
    std::vector<std::string> cols(names, names + ncols);
    CsvWriter w(path, cols);
    for (int r = 0; r < nrows; ++r)
      w.write_row(std::vector<double>(values + (size_t)r * ncols, values + (size_t)(r + 1) * ncols));
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

// read_csv (csv.hpp:88-112): rows x cols values, returns rows or -1
int ref_csv_read(const char* path, int max_values, double* values, int* ncols) {
  try {
    const CsvTable t = read_csv(path);
    *ncols = (int)t.columns.size();
    int k = 0;
    for (const auto& r : t.rows)
      for (double v : r)
        if (k < max_values) values[k++] = v;
    return (int)t.rows.size();
  } catch (const std::exception&) {
    return -1;
  }
}

const char* ref_last_error() { return g_err; }

// ---------------------------------------------------------------- units ---
double ref_units_tau(double dx, double dt, double rho, double nu) {
  return make_units(dx, dt, rho, nu).tau();
}
int ref_units_validate(double dx, double dt, double rho, double nu) {
  try {
    make_units(dx, dt, rho, nu).validate();
    return 0;
  } catch (const InputError& e) {
    std::snprintf(g_err, sizeof g_err, "%s", e.what());
    return 1;
  }
}

// ------------------------------------------------------------------ rng ---
void ref_rng_uniform(uint64_t seed, int64_t n, double* out) {
  Rng r(seed);
  for (int64_t k = 0; k < n; ++k) out[k] = r.uniform();
}
void ref_rng_normal(uint64_t seed, int64_t n, double* out) {
  Rng r(seed);
  for (int64_t k = 0; k < n; ++k) out[k] = r.normal();
}

// -------------------------------------------------------------- session ---
// mode: 0 = Periodic, 1 = OpenExtrapolated (lattice.hpp:53-56)
// kernel: 0 = Peskin4, 1 = Roma3; wall: 0 = Slip, 1 = NoSlip
// frame_mode: 0 None, 1 Translation, 2 TranslationYaw, 3 Full
void* ref_session_create(int nx, int ny, int nz, double dx, double dt, double rho, double nu,
                         int periodic, int kernel, int wall, int frame_mode) {
  try {
    auto s = std::make_unique<RefSession>();
    s->dims = {nx, ny, nz};
    s->units = make_units(dx, dt, rho, nu);
    s->grid = lbm::LatticeGrid(s->dims, s->units,
                               periodic ? lbm::BoundaryMode::Periodic
                                        : lbm::BoundaryMode::OpenExtrapolated);
    s->force.resize(s->dims);
    s->macro.resize(s->dims);
    s->kernel.family = kernel == 0 ? ib::IBKernel::Family::Peskin4 : ib::IBKernel::Family::Roma3;
    s->wall = wall == 0 ? ib::WallCondition::Slip : ib::WallCondition::NoSlip;
    s->frame_mode = static_cast<frame::FollowMode>(frame_mode);
    return s.release();
  } catch (const std::exception& e) {
    std::snprintf(g_err, sizeof g_err, "%s", e.what());
    return nullptr;
  }
}

void ref_session_destroy(void* h) { delete static_cast<RefSession*>(h); }

int64_t ref_n_cells(void* h) { return static_cast<int64_t>(static_cast<RefSession*>(h)->grid.n_cells()); }

void ref_reset_rest(void* h) { static_cast<RefSession*>(h)->grid.reset_to_rest(); }

/// Whole distribution set, direction-major f[i*n + cell] (lattice.hpp:89-90).
void ref_set_f(void* h, const double* f) {
  auto* s = static_cast<RefSession*>(h);
  std::memcpy(s->grid.front().data(), f, sizeof(double) * s->grid.front().size());
}
void ref_get_f(void* h, double* f) {
  auto* s = static_cast<RefSession*>(h);
  std::memcpy(f, s->grid.front().data(), sizeof(double) * s->grid.front().size());
}

/// LatticeGrid::initialize (lattice.hpp:107-116) from per-cell rho[n], u[3n].
void ref_initialize(void* h, const double* rho, const double* u) {
  auto* s = static_cast<RefSession*>(h);
  const int nx = s->dims[0], ny = s->dims[1];
  s->grid.initialize(
      [&](int x, int y, int z) { return rho[x + static_cast<size_t>(nx) * (y + static_cast<size_t>(ny) * z)]; },
      [&](int x, int y, int z) {
        const size_t c = x + static_cast<size_t>(nx) * (y + static_cast<size_t>(ny) * z);
        return Vec3(u[3 * c], u[3 * c + 1], u[3 * c + 2]);
      });
}

/// Body force field, AoS Vec3 per cell (lattice.hpp:145-154).
void ref_set_force(void* h, const double* F) {
  auto* s = static_cast<RefSession*>(h);
  for (size_t c = 0; c < s->force.F.size(); ++c) s->force.F[c] = Vec3(F[3 * c], F[3 * c + 1], F[3 * c + 2]);
}
void ref_get_force(void* h, double* F) {
  auto* s = static_cast<RefSession*>(h);
  for (size_t c = 0; c < s->force.F.size(); ++c) put3(F + 3 * c, s->force.F[c]);
}

/// lbm::collide_and_stream (solver.hpp:103-178).
void ref_collide_and_stream(void* h, int* finite, double* min_f) {
  auto* s = static_cast<RefSession*>(h);
  const auto st = lbm::collide_and_stream(s->grid, s->force);
  *finite = st.finite ? 1 : 0;
  *min_f = st.min_f;
}

/// lbm::apply_open_boundary (solver.hpp:65-97) on the front buffer.
void ref_apply_open_boundary(void* h) { lbm::apply_open_boundary(static_cast<RefSession*>(h)->grid); }

/// lbm::macroscopic_into (solver.hpp:25-51) with the current force field.
int ref_macroscopic(void* h, double* rho, double* u) {
  auto* s = static_cast<RefSession*>(h);
  lbm::macroscopic_into(s->grid, s->force, s->macro);
  for (size_t c = 0; c < s->macro.rho.size(); ++c) {
    rho[c] = s->macro.rho[c];
    put3(u + 3 * c, s->macro.u[c]);
  }
  return s->macro.n_nonpositive_rho;
}

double ref_total_mass(void* h) { return lbm::total_mass(static_cast<RefSession*>(h)->grid); }
void ref_total_momentum(void* h, double* p) { put3(p, lbm::total_momentum(static_cast<RefSession*>(h)->grid)); }
double ref_kinetic_energy(void* h) { return lbm::kinetic_energy(static_cast<RefSession*>(h)->macro); }

/// Frame state in world terms (frame.hpp:13-43); quaternion (w,x,y,z).
void ref_set_frame(void* h, const double* p, const double* pd, const double* pdd, const double* q,
                   const double* omega, const double* alpha) {
  auto* s = static_cast<RefSession*>(h);
  s->fs.p = v3(p);
  s->fs.pd = v3(pd);
  s->fs.pdd = v3(pdd);
  s->fs.rot = Quat(q[0], q[1], q[2], q[3]);
  s->fs.omega = v3(omega);
  s->fs.alpha = v3(alpha);
}
void ref_get_frame_p(void* h, double* p) { put3(p, static_cast<RefSession*>(h)->fs.p); }
void ref_frame_rotation(void* h, double* r9) {
  const Mat3 r = static_cast<RefSession*>(h)->fs.rotation();
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r9[3 * i + j] = r(i, j);
}

/// frame::recenter (frame.hpp:132-154).
void ref_recenter(void* h, const int* shift) {
  auto* s = static_cast<RefSession*>(h);
  frame::recenter(s->grid, s->fs, Index3{shift[0], shift[1], shift[2]});
}

/// The fluid half of CoupledSession::step (session.hpp:94-166) for ONE body
/// whose world-frame marker state is supplied by the caller instead of by
/// robot::update_samples. Outputs: per-marker world force (N) and validity,
/// the CouplingStats sums (session.hpp:141-143: fluid force, power with the
/// caller's velocities), the collide status and the non-positive rho count.
/// n_bodies markers sets are concatenated; body_offsets has n_bodies+1 entries.
int ref_session_step(void* h, int n_bodies, const int64_t* body_offsets, const double* points,
                     const double* velocities, const double* normals, const double* areas,
                     double* force_world, int* valid, double* stats /*n_bodies*7*/, int* finite,
                     double* min_f) {
  auto* S = static_cast<RefSession*>(h);
  const Real dt = S->units.dt_phys;
  const Real dx = S->units.dx;
  const auto& fs = S->fs;
  const Mat3 r_frame = fs.rotation();
  int nonpos = 0;

  S->force.clear();
  lbm::macroscopic_into(S->grid, S->force, S->macro);
  nonpos = S->macro.n_nonpositive_rho;

  for (int b = 0; b < n_bodies; ++b) {
    const int64_t off = body_offsets[b];
    const size_t n = static_cast<size_t>(body_offsets[b + 1] - off);
    S->sample_force_world.assign(n, Vec3::Zero());
    S->sample_valid.assign(n, 0);
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < static_cast<long long>(n); ++i) {
      const size_t g = off + i;
      const Vec3 x_frame = fs.world_to_frame_point(v3(points + 3 * g));
      const Vec3 x_lat = frame_to_lattice(*S, x_frame);
      if (!ib::marker_in_bounds(S->kernel, S->dims, x_lat)) continue;
      S->sample_valid[i] = 1;
      const Vec3 u_f_frame =
          S->units.vel_to_physical(ib::interpolate_velocity(S->macro, S->kernel, x_lat));
      const Vec3 u_b_frame = fs.body_velocity_to_frame(x_frame, v3(velocities + 3 * g));
      const Vec3 n_frame = r_frame.transpose() * v3(normals + 3 * g);
      S->sample_force_world[i] =
          r_frame * ib::direct_forcing(u_b_frame, u_f_frame, n_frame, S->units.rho_phys,
                                       areas[g], dx, dt, S->wall);
    }
    const Real force_to_lattice = dt * dt / (S->units.rho_phys * dx * dx * dx * dx);
    Vec3 tot_fluid = Vec3::Zero(), tot_body = Vec3::Zero();
    Real power = 0.0;
    int oob = 0;
    for (size_t i = 0; i < n; ++i) {
      const size_t g = off + i;
      valid[g] = S->sample_valid[i];
      put3(force_world + 3 * g, S->sample_force_world[i]);
      if (!S->sample_valid[i]) {
        ++oob;
        continue;
      }
      const Vec3& f_world = S->sample_force_world[i];
      const Vec3 f_frame = r_frame.transpose() * f_world;
      const Vec3 x_lat = frame_to_lattice(*S, fs.world_to_frame_point(v3(points + 3 * g)));
      ib::spread_force(S->force, S->kernel, x_lat, f_frame * force_to_lattice);
      tot_fluid += f_world;
      tot_body -= f_world;
      power += (-f_world).dot(v3(velocities + 3 * g));
    }
    put3(stats + 7 * b, tot_fluid);
    put3(stats + 7 * b + 3, tot_body);
    stats[7 * b + 6] = power;
    (void)oob;
  }

  if (S->frame_mode != frame::FollowMode::None) {
    const Real acc_to_lattice = dt * dt / dx;
    const Index3 d = S->dims;
#pragma omp parallel for schedule(static)
    for (int k = 0; k < d[2]; ++k) {
      for (int j = 0; j < d[1]; ++j) {
        for (int i = 0; i < d[0]; ++i) {
          const size_t c = S->grid.cell_index(i, j, k);
          const Vec3 x_frame = cell_frame_position(*S, i, j, k);
          const Vec3 u_frame = S->units.vel_to_physical(S->macro.u[c]);
          const Vec3 a = frame::virtual_force(fs, x_frame, u_frame);
          S->force.F[c] += S->macro.rho[c] * acc_to_lattice * a;
        }
      }
    }
  }

  const auto status = lbm::collide_and_stream(S->grid, S->force);
  *finite = status.finite ? 1 : 0;
  *min_f = status.min_f;
  return nonpos;
}

/// Marker lattice coordinates as the session computes them
/// (frame_to_lattice(world_to_frame_point(x)), session.hpp:115-116).
void ref_session_marker_xlat(void* h, int64_t n, const double* points, double* xlat) {
  auto* S = static_cast<RefSession*>(h);
  for (int64_t i = 0; i < n; ++i)
    put3(xlat + 3 * i, frame_to_lattice(*S, S->fs.world_to_frame_point(v3(points + 3 * i))));
}

/// Bare macroscopic fields from the last session step (session.hpp:95-96).
void ref_get_macro(void* h, double* rho, double* u) {
  auto* s = static_cast<RefSession*>(h);
  for (size_t c = 0; c < s->macro.rho.size(); ++c) {
    rho[c] = s->macro.rho[c];
    put3(u + 3 * c, s->macro.u[c]);
  }
}

// ------------------------------------------------------------------- IB ---
double ref_phi(int kernel, double r) {
  ib::IBKernel k{kernel == 0 ? ib::IBKernel::Family::Peskin4 : ib::IBKernel::Family::Roma3};
  return k.phi(r);
}
void ref_range(int kernel, double x, int* lo, int* hi) {
  ib::IBKernel k{kernel == 0 ? ib::IBKernel::Family::Peskin4 : ib::IBKernel::Family::Roma3};
  k.range(x, *lo, *hi);
}
int ref_marker_in_bounds(int kernel, const int* dims, const double* x) {
  ib::IBKernel k{kernel == 0 ? ib::IBKernel::Family::Peskin4 : ib::IBKernel::Family::Roma3};
  return ib::marker_in_bounds(k, Index3{dims[0], dims[1], dims[2]}, v3(x)) ? 1 : 0;
}
/// ib::interpolate_velocity (coupling.hpp:27-48) over a caller u field [3n].
void ref_interpolate(int kernel, const int* dims, const double* ufield, int n, const double* x,
                     double* out) {
  ib::IBKernel k{kernel == 0 ? ib::IBKernel::Family::Peskin4 : ib::IBKernel::Family::Roma3};
  lbm::FluidMacro m;
  m.resize(Index3{dims[0], dims[1], dims[2]});
  for (size_t c = 0; c < m.u.size(); ++c) m.u[c] = v3(ufield + 3 * c);
  for (int i = 0; i < n; ++i) put3(out + 3 * i, ib::interpolate_velocity(m, k, v3(x + 3 * i)));
}
/// ib::spread_force (coupling.hpp:52-71), markers in ascending order into F [3n].
void ref_spread(int kernel, const int* dims, int n, const double* x, const double* f, double* F) {
  ib::IBKernel k{kernel == 0 ? ib::IBKernel::Family::Peskin4 : ib::IBKernel::Family::Roma3};
  lbm::BodyForceField field;
  field.resize(Index3{dims[0], dims[1], dims[2]});
  for (size_t c = 0; c < field.F.size(); ++c) field.F[c] = v3(F + 3 * c);
  for (int i = 0; i < n; ++i) ib::spread_force(field, k, v3(x + 3 * i), v3(f + 3 * i));
  for (size_t c = 0; c < field.F.size(); ++c) put3(F + 3 * c, field.F[c]);
}
/// ib::direct_forcing (coupling.hpp:80-85).
void ref_direct_forcing(const double* ub, const double* uf, const double* n, double rho,
                        double area, double h, double dt, int wall, double* out) {
  put3(out, ib::direct_forcing(v3(ub), v3(uf), v3(n), rho, area, h, dt,
                               wall == 0 ? ib::WallCondition::Slip : ib::WallCondition::NoSlip));
}

// ---------------------------------------------------------------- frame ---
/// frame::virtual_force (frame.hpp:47-53).
void ref_virtual_force(const double* q, const double* pdd, const double* omega,
                       const double* alpha, const double* x, const double* u, double* out) {
  frame::FrameState f;
  f.rot = Quat(q[0], q[1], q[2], q[3]);
  f.pdd = v3(pdd);
  f.omega = v3(omega);
  f.alpha = v3(alpha);
  put3(out, frame::virtual_force(f, v3(x), v3(u)));
}

/// frame::FrameFollower (frame.hpp:70-125).
void* ref_follower_create(int mode, double tc) {
  return new frame::FrameFollower(static_cast<frame::FollowMode>(mode), tc);
}
void ref_follower_destroy(void* h) { delete static_cast<frame::FrameFollower*>(h); }
void ref_follower_reset(void* h, const double* p, double yaw) {
  static_cast<frame::FrameFollower*>(h)->reset(v3(p), yaw);
}
void ref_follower_step(void* h, const double* target_p, const double* target_q, double dt) {
  static_cast<frame::FrameFollower*>(h)->step(
      v3(target_p), Quat(target_q[0], target_q[1], target_q[2], target_q[3]), dt);
}
/// state out: p, pd, pdd, q(w,x,y,z), omega, alpha, euler(r,p,y)  = 22 doubles
void ref_follower_state(void* h, double* out) {
  const auto& f = static_cast<frame::FrameFollower*>(h)->state();
  put3(out, f.p);
  put3(out + 3, f.pd);
  put3(out + 6, f.pdd);
  out[9] = f.rot.w();
  out[10] = f.rot.x();
  out[11] = f.rot.y();
  out[12] = f.rot.z();
  put3(out + 13, f.omega);
  put3(out + 16, f.alpha);
  put3(out + 19, f.euler());
}
void ref_quat_exp(const double* w, double* q) {
  const Quat r = quat_exp(v3(w));
  q[0] = r.w();
  q[1] = r.x();
  q[2] = r.y();
  q[3] = r.z();
}

}  // extern "C"
