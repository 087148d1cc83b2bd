/* fsg.h -- C ABI of the B200-native FishGym IB-LBM hot path.
 *
 * This is the drop-in boundary.  The reference (FishGym,
 * /root/reference/proj/include/fishsim) exposes the path as a header-only
 * C++ API with no FFI; each entry point below replaces one reference call,
 * cited as file:line.  A C++ wrapper with the reference's class shapes
 * (CoupledSession, LatticeGrid, FrameFollower ...) sits on top of this ABI in
 * include/fishgym_b200/session.hpp; Python binds it with ctypes
 * (paper_2206_01683_b200/_abi.py).
 *
 * Conventions (identical to the reference):
 *   cell index    c = x + nx*(y + ny*z)                    lattice.hpp:83-87
 *   distributions f[i*n + c], i in D3Q19 order             lattice.hpp:17-38, :89-90
 *   vector fields AoS, v[3*c + k]                          lattice.hpp:129-154
 *   lattice units; marker state in SI world coordinates    session.hpp:113-126
 * All host pointers are plain C arrays owned by the caller.  Every call
 * returns FSG_OK (0) or an error code; fsg_last_error() gives a
 * thread-local message.  Invalid configuration -> FSG_EINPUT (the
 * reference throws InputError); runtime instability is NOT an error, it is
 * reported in fsg_status (solver.hpp:13-20, backend.hpp:37-40).
 * One session = one device + one CUDA stream; a session is not thread-safe
 * (SPEC.md:113); independent sessions may run concurrently.
 */
#ifndef FSG_H
#define FSG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSG_ABI_VERSION 1

enum { FSG_OK = 0, FSG_EINPUT = 1, FSG_ECUDA = 2, FSG_ESTATE = 3 };

/* lattice.hpp:53-56 */
enum { FSG_BOUNDARY_PERIODIC = 0, FSG_BOUNDARY_OPEN = 1 };
/* kernel.hpp:15-20 */
enum { FSG_KERNEL_PESKIN4 = 0, FSG_KERNEL_ROMA3 = 1 };
/* coupling.hpp:73-76 */
enum { FSG_WALL_SLIP = 0, FSG_WALL_NOSLIP = 1 };
/* frame.hpp:55 */
enum { FSG_FRAME_NONE = 0, FSG_FRAME_TRANSLATION = 1, FSG_FRAME_TRANSLATION_YAW = 2, FSG_FRAME_FULL = 3 };
/* storage/arithmetic of the distribution set:
 *   FP32 : fp32 storage of f - w_i, fp32 deviation arithmetic (throughput mode, 152 B/cell)
 *   FP64 : fp64 storage and the reference's fp64 operation order, no FMA
 *          contraction (parity mode: bit-identical to the reference)            */
enum { FSG_PRECISION_FP32 = 0, FSG_PRECISION_FP64 = 1 };

/* SessionConfig (session.hpp:12-24) + UnitMap (units.hpp:18-23) +
 * LatticeGrid ctor arguments (lattice.hpp:63-74). */
typedef struct {
  int dims[3];        /* cells per axis, each >= 8 (lattice.hpp:66-67)          */
  double dx;          /* m per cell                                             */
  double dt;          /* s per lattice step                                     */
  double rho;         /* kg/m^3 mapped to lattice density 1                     */
  double nu;          /* m^2/s ; tau = 3 nu dt/dx^2 + 1/2 must lie in (0.5,1.5]  */
  int boundary;       /* FSG_BOUNDARY_*  (CoupledSession uses OPEN)             */
  int kernel;         /* FSG_KERNEL_*                                           */
  int wall;           /* FSG_WALL_*                                             */
  int frame_mode;     /* FSG_FRAME_*                                            */
  int precision;      /* FSG_PRECISION_*                                        */
  int device;         /* CUDA device ordinal                                    */
  int max_markers;    /* marker capacity (all bodies), 0 -> 65536               */
  /* z-slab decomposition; a single-GPU session uses
   * z_offset = 0 and nz_global = dims[2].  dims[2] is the LOCAL slab depth. */
  int z_offset;
  int nz_global;
} fsg_config;

/* StepStatus (solver.hpp:13-20) + StepOutcome (backend.hpp:37-40). */
typedef struct {
  int finite;                 /* every cell had finite rho + |u|^2             */
  double min_f;               /* min post-collision population                 */
  int n_nonpositive_rho;      /* FluidMacro::n_nonpositive_rho (solver.hpp:42) */
  int out_of_bounds_markers;  /* session.hpp:130-134                           */
  int stable;                 /* finite && min_f > -1e-3 && nonpos == 0        */
} fsg_status;

/* FrameState (frame.hpp:13-20), world frame; q = (w, x, y, z). */
typedef struct {
  double p[3], pd[3], pdd[3], q[4], omega[3], alpha[3];
} fsg_frame_state;

typedef struct fsg_session fsg_session;

const char* fsg_last_error(void);
int fsg_abi_version(void);
/* Default config = SessionConfig defaults (session.hpp:12-24). */
void fsg_config_default(fsg_config* cfg);
/* UnitMap::tau (units.hpp:25). */
double fsg_tau(double dx, double dt, double nu);

/* CoupledSession(cfg) (session.hpp:31-40): validates units (units.hpp:56-68),
 * dims >= 8, allocates the A/B distribution pair in HBM at rest. */
int fsg_create(const fsg_config* cfg, fsg_session** out);
int fsg_destroy(fsg_session* s);
/* the session's CUDA stream (cudaStream_t), for event timing / interop */
void* fsg_stream(fsg_session* s);

/* ---- LatticeGrid (lattice.hpp:60-126) ---------------------------------- */
int fsg_reset_rest(fsg_session* s);                                   /* :98-104  */
int fsg_initialize(fsg_session* s, const double* rho, const double* u); /* :107-116 */
int fsg_set_f(fsg_session* s, const double* f);   /* front() assignment, f[19*n]     */
int fsg_get_f(fsg_session* s, double* f);         /* front() readback (post-stream)  */

/* ---- lbm::solver (solver.hpp) ------------------------------------------ */
/* BodyForceField used by fsg_collide_and_stream / fsg_macroscopic; NULL clears. */
int fsg_set_force(fsg_session* s, const double* F);
int fsg_collide_and_stream(fsg_session* s, fsg_status* st);            /* :103-178 */
int fsg_macroscopic(fsg_session* s, double* rho, double* u, int* n_nonpositive); /* :25-51 */
int fsg_total_mass(fsg_session* s, double* mass);                       /* :181-187 */
int fsg_total_momentum(fsg_session* s, double* p3);                     /* :189-200 */

/* ---- frame (frame.hpp) ---------------------------------------------------- */
int fsg_set_frame(fsg_session* s, const fsg_frame_state* fs);
int fsg_get_frame(fsg_session* s, fsg_frame_state* fs);
/* frame::recenter (frame.hpp:132-154): shifts the lattice by an integer cell
 * offset and advances the frame origin by R*shift*dx. */
int fsg_recenter(fsg_session* s, const int shift[3]);

/* frame::FrameFollower (frame.hpp:70-125): the critically damped tracker of
 * the robot base that produces the frame state fed to fsg_set_frame.  Host
 * code (no device), fp64, bit-identical to the reference's.  mode: FSG_FRAME_*
 * (follow_mode), time_constant in s (wn = 1/time_constant; 0.2 s default). */
typedef struct fsg_follower fsg_follower;
int fsg_follower_create(int mode, double time_constant, fsg_follower** out);
int fsg_follower_destroy(fsg_follower* f);
int fsg_follower_reset(fsg_follower* f, const double p[3], double yaw);             /* :81-87 */
int fsg_follower_step(fsg_follower* f, const double target_p[3], const double target_q[4],
                      double dt);                                                     /* :90-119 */
int fsg_follower_state(const fsg_follower* f, fsg_frame_state* out);
/* restore a state (e.g. the origin shift of fsg_recenter, a checkpoint) */
int fsg_follower_set_state(fsg_follower* f, const fsg_frame_state* in);
/* CoupledSession::center_frame_on_robot (session.hpp:210-221): reset to the
 * robot base position with its yaw (0 in TRANSLATION mode; origin in NONE) */
int fsg_follower_center(fsg_follower* f, const double base_p[3], const double base_q[4]);

/* ---- coupled step (session.hpp:87-198, fluid half :94-166) -------------- */
/* Marker state for this step, world frame SI (what robot::update_samples
 * produces, sampling.hpp:307-322): n_bodies bodies, body b owns markers
 * [body_offsets[b], body_offsets[b+1]).  points/velocities/normals are [3*m],
 * areas [m].  Host pointers; copied to HBM. */
int fsg_set_markers(fsg_session* s, int n_bodies, const int64_t* body_offsets,
                    const double* points, const double* velocities, const double* normals,
                    const double* areas);
/* Same, but the four arrays are DEVICE pointers already resident in HBM. */
int fsg_set_markers_device(fsg_session* s, int n_bodies, const int64_t* body_offsets,
                           const double* d_points, const double* d_velocities,
                           const double* d_normals, const double* d_areas);
/* One coupled fluid step: bare moments, marker interpolation + direct
 * forcing, ordered spreading, virtual force, collide+stream+open BC.
 * Synchronous: returns the StepStatus. */
int fsg_step(fsg_session* s, fsg_status* st);
/* Enqueue the step on the session stream without waiting (status available
 * through fsg_last_status after a later sync). */
int fsg_step_async(fsg_session* s);
int fsg_last_status(fsg_session* s, fsg_status* st);
/* Per-marker world force on the FLUID (N) and validity of the last step
 * (session.hpp:124-125, :130); CouplingStats per body (coupling.hpp:88-93):
 * stats[7*b] = {force_on_fluid[3], force_on_body[3], power_on_body}. */
int fsg_get_marker_forces(fsg_session* s, double* force_world, int* valid, double* stats);
/* Bare macroscopic fields of the last step (CoupledSession::macro(), session.hpp:95-96). */
int fsg_get_macro(fsg_session* s, double* rho, double* u);
/* BodyForceField of the last step, IB + virtual force, AoS (session.hpp:148-163).
 * fp64 sessions: the field the collision used.  fp32 sessions: with force
 * capture on (fsg_set_force_capture) the field the throughput collision
 * kernel itself consumed, captured cell by cell; otherwise a diagnostic
 * rebuild from the step's stencil records. */
int fsg_get_force(fsg_session* s, double* F);
/* Diagnostic (fp32 coupled steps): have the collision kernel store the body
 * force it consumes (fixed-point IB band decoded + virtual force, 12 B per
 * cell per step) for fsg_get_force.  Off by default. */
int fsg_set_force_capture(fsg_session* s, int on);
/* Integer stencil sets of the last step, per marker: lo[3], hi[3] (kernel.hpp:36-40). */
int fsg_get_stencils(fsg_session* s, int* lo_hi);

/* ---- skinned bodies on the device -------------------
 * Per-step marker refresh and Jacobian-transpose force reduction of the
 * robot side of CoupledSession::step (session.hpp:103-144), so only the
 * per-link pose goes up and only tau_ext + CouplingStats come back:
 *   robot::update_samples        (sampling.hpp:307-322): LBS of points,
 *       skin_point / skin_point_velocity (skinning.hpp:105-126) and normals;
 *   robot::accumulate_skinned_force (skinning.hpp:147-156) ->
 *       accumulate_point_force (dynamics.hpp:216-233), called with -f_world
 *       per valid marker in ascending order (session.hpp:129-140);
 *   CouplingStats (coupling.hpp:88-93, session.hpp:141-143).
 * Forward kinematics and BoneTransforms::of stay with the caller (host, per
 * link); fsg_set_pose takes their results. */
#define FSG_SKIN_MAX_LINKS 12 /* the reference eel: 11 links (model_builder.hpp:234-249) */
#define FSG_SKIN_MAX_BODIES 4
#define FSG_SKIN_MAX_WEIGHTS 4 /* nonzero blend weights per marker */

/* Skeleton topology (skeleton.hpp:16-93). */
typedef struct {
  int n_links;                          /* <= FSG_SKIN_MAX_LINKS                     */
  int floating_base;                    /* links[0].joint == Free (skeleton.hpp:72)  */
  int n_dofs;                           /* Skeleton::n_dofs()                        */
  int parent[FSG_SKIN_MAX_LINKS];       /* links[i].parent (-1 for the root)         */
  int dof_index[FSG_SKIN_MAX_LINKS];    /* Skeleton::dof_index(i), -1: no revolute dof */
  double axis[FSG_SKIN_MAX_LINKS][3];   /* links[i].axis.normalized() (revolute)     */
} fsg_skeleton;

/* Per-step pose of one body: BoneTransforms::of (skinning.hpp:85-102) and the
 * KinematicsCache fields the path reads (dynamics.hpp:14-21); row-major. */
typedef struct {
  double bone_R[FSG_SKIN_MAX_LINKS][9];
  double bone_t[FSG_SKIN_MAX_LINKS][3];
  double R_world[FSG_SKIN_MAX_LINKS][9];
  double p_world[FSG_SKIN_MAX_LINKS][3];
  double v_origin_world[FSG_SKIN_MAX_LINKS][3];
  double omega_world[FSG_SKIN_MAX_LINKS][3];
} fsg_body_pose;

/* Register skinned bodies (SurfaceSamples, sampling.hpp): body b owns
 * markers [body_offsets[b], body_offsets[b+1]); rest_points/rest_normals
 * [3m] (base at identity), areas [m], weights: for each marker, n_links(b)
 * blend weights (rows sum to 1; at most FSG_SKIN_MAX_WEIGHTS nonzero).
 * Replaces fsg_set_markers: every later step skins the markers on the device
 * from the pose set by fsg_set_pose (until fsg_set_markers* is called). */
int fsg_set_skin(fsg_session* s, int n_bodies, const int64_t* body_offsets,
                 const fsg_skeleton* skeletons, const double* rest_points,
                 const double* rest_normals, const double* weights, const double* areas);
/* This step's pose of every skinned body (n_bodies entries). */
int fsg_set_pose(fsg_session* s, const fsg_body_pose* poses);
/* Of the last step: tau_ext of every body (concatenated, n_dofs(b) each;
 * session.hpp:107, :139-140) and CouplingStats stats[7*b] as in
 * fsg_get_marker_forces.  Either pointer may be NULL. */
int fsg_get_body_wrench(fsg_session* s, double* tau_ext, double* stats);
/* The robot loop's whole per-step exchange in one call: fsg_set_frame (fs
 * may be NULL: keep the frame), fsg_set_pose, fsg_step (synchronous status),
 * fsg_get_body_wrench. */
int fsg_step_skinned(fsg_session* s, const fsg_frame_state* fs, const fsg_body_pose* poses,
                     fsg_status* st, double* tau_ext, double* stats);
/* Marker state the last step used (world frame; skinned or uploaded). */
int fsg_get_markers(fsg_session* s, double* points, double* velocities, double* normals);

/* ---- empirical drag backend, batched ----------------
 * EmpiricalBackend::step (empirical.hpp:74-100) for n_envs envs of one robot
 * each, up to the robot integration: device-side skinning of the samples
 * (update_samples), surface_force F = -k (n.v) n A on advancing patches
 * (empirical.hpp:25-30), tau_ext += J^T F (accumulate_skinned_force) and
 * CouplingStats (force on body, power).  precision FSG_PRECISION_FP64: the
 * reference's serial order, bit-identical; FSG_PRECISION_FP32: fp64
 * arithmetic with a deterministic fixed-point (2^-44) reduction.  Errors:
 * fsg_drag_last_error(). */
typedef struct fsg_drag fsg_drag;
const char* fsg_drag_last_error(void);
int fsg_drag_create(int n_envs, double k, int precision, int device, fsg_drag** out);
int fsg_drag_destroy(fsg_drag* d);
/* env's robot: SurfaceSamples (rest points/normals [3m], weights [m][n_links], areas [m]) */
int fsg_drag_set_skin(fsg_drag* d, int env, const fsg_skeleton* skeleton, int m,
                      const double* rest_points, const double* rest_normals,
                      const double* weights, const double* areas);
int fsg_drag_set_pose(fsg_drag* d, int env, const fsg_body_pose* pose);
/* every env's pose at once (n_envs entries) */
int fsg_drag_set_poses(fsg_drag* d, const fsg_body_pose* poses);
/* one step of every env: tau_ext (concatenated n_dofs per env) and
 * stats[7*env] = {force_on_fluid[3] (0), force_on_body[3], power_on_body} */
int fsg_drag_step(fsg_drag* d, double* tau_ext, double* stats);

/* ---- articulated robot dynamics, batched -------------
 * The robot half of CoupledSession::step (session.hpp:169-175) for n_envs
 * robots of one Skeleton on the device, one thread per env in fp64:
 *   hydro = robot::buoyancy_gravity_forces(kc(state), bladder, rho, g_hydro)
 *                                                    (dynamics.hpp:237-255)
 *   robot::integrate(state, actuation, tau_ext + hydro, dt, substeps, gravity)
 *                                                    (dynamics.hpp:259-289)
 * with forward_kinematics / mass_matrix (CRBA) / bias_forces (RNEA) /
 * internal_forces / joint_limit_forces / LLT solve (dynamics.hpp:23-212),
 * and the new pose for device skinning (fsg_dyn_poses: forward_kinematics +
 * BoneTransforms::of, skinning.hpp:85-102).  Results agree with the fp64
 * restatement to rounding (libm vs device sin/cos: rel <= 1e-12 per step).
 * Errors: fsg_dyn_last_error() (Skeleton::validate messages, InputError);
 * a mass matrix that is not positive definite (NumericalError in the
 * reference, dynamics.hpp:208-210) sets FSG_DYN_NOT_SPD in the env's flags
 * and stops that env at the failing substep: its state keeps the substeps
 * completed before it (as the reference's integrate throwing mid-loop). */
#define FSG_DYN_MAX_LINKS 12 /* eel: 11 links, 16 dofs */
#define FSG_DYN_MAX_DOFS (6 + FSG_DYN_MAX_LINKS)
enum { FSG_JOINT_FREE = 0, FSG_JOINT_REVOLUTE = 1, FSG_JOINT_FIXED = 2 };
enum { FSG_DYN_CLAMPED = 1, FSG_DYN_NOT_SPD = 2, FSG_DYN_NONFINITE = 4 };

/* robot::Link (skeleton.hpp:16-36); matrices row-major */
typedef struct {
  int parent; /* -1 for the root */
  int joint;  /* FSG_JOINT_* */
  double joint_origin[3];
  double joint_rotation[9];
  double axis[3];
  double mass;
  double com[3];
  double inertia_com[9];
  double stiffness, damping, q_rest, limit_lo, limit_hi, torque_limit;
  double displaced_volume;
  double volume_centroid[3];
} fsg_link;

/* robot::Skeleton + its Bladder (skeleton.hpp:38-93) */
typedef struct {
  int n_links;
  fsg_link links[FSG_DYN_MAX_LINKS];
  double bladder_volume, bladder_volume_min, bladder_volume_max, bladder_rate_bound;
  double bladder_centroid[3];
} fsg_robot;

/* robot::JointState (skeleton.hpp:138-150); quaternion (w, x, y, z) */
typedef struct {
  double base_pos[3];
  double base_quat[4];
  double q[FSG_DYN_MAX_LINKS];
  double v[FSG_DYN_MAX_DOFS];
  double qdd[FSG_DYN_MAX_DOFS];
} fsg_joint_state;

typedef struct fsg_dyn fsg_dyn;
const char* fsg_dyn_last_error(void);
/* validates the skeleton as Skeleton::validate; every env starts at
 * JointState::zero with the robot's bladder */
int fsg_dyn_create(const fsg_robot* robot, int n_envs, int device, fsg_dyn** out);
int fsg_dyn_destroy(fsg_dyn* d);
int fsg_dyn_n_dofs(const fsg_dyn* d);
int fsg_dyn_n_joints(const fsg_dyn* d);
int fsg_dyn_set_state(fsg_dyn* d, const fsg_joint_state* states); /* n_envs */
int fsg_dyn_get_state(fsg_dyn* d, fsg_joint_state* states);
/* Bladder::apply_change per env (skeleton.hpp:48-51, Backend::change_bladder);
 * volumes (nullable) receives the new volumes */
int fsg_dyn_change_bladder(fsg_dyn* d, const double* dv, double* volumes);
/* one robot step of every env (host arrays): actuation [n_envs * n_joints],
 * tau_ext [n_envs * n_dofs] (NULL: zero), flags [n_envs] (nullable).
 * g_hydro: gravity of buoyancy_gravity_forces (NULL: no hydrostatics);
 * gravity: integrate's gravity argument (NULL: zero). */
int fsg_dyn_step(fsg_dyn* d, const double* actuation, const double* tau_ext, double rho_fluid,
                 const double* g_hydro, double dt, int substeps, const double* gravity,
                 int* flags);
/* the same with device pointers, stream-ordered on the handle's stream */
int fsg_dyn_step_device(fsg_dyn* d, const double* d_actuation, const double* d_tau_ext,
                        double rho_fluid, const double* g_hydro, double dt, int substeps,
                        const double* gravity, int* d_flags);
/* parity probes: mass_matrix (row-major nd x nd per env) and bias_forces (nd)
 * at the current state; either pointer may be NULL */
int fsg_dyn_mass_matrix(fsg_dyn* d, const double* gravity, double* M, double* bias);
/* the current state's pose of every env for fsg_set_pose / fsg_drag_set_poses
 * (rest_R [n_links*9], rest_p [n_links*3]: BoneTransforms rest pose) */
int fsg_dyn_poses(fsg_dyn* d, const double* rest_R, const double* rest_p, fsg_body_pose* poses);
/* the rest pose (RestPose::of) the device-side poses of fsg_batch_step_dynamic use */
int fsg_dyn_set_rest(fsg_dyn* d, const double* rest_R, const double* rest_p);

/* ---- output formats -----------------------------------
 * fsg_snapshot_begin enqueues the bare moments of the state the last step
 * read (CoupledSession::macro(), session.hpp:95-96) into a snapshot buffer and
 * copies it to pinned host memory on the copy stream: later steps proceed
 * while it travels.  fsg_snapshot_wait returns it (rho [n], u [3n], lattice
 * units, cell order).  fsg_write_vtk writes the latest snapshot as
 * lbm::write_vtk (vtk.hpp:15-38) does, byte for byte; fsg_write_vtk_fields
 * writes given fields.  fsg_csv_* is CsvWriter (csv.hpp:27-66) with
 * format_full's %.17g round-trip formatting (csv.hpp:18-22).  Errors of the
 * host-only writers: fsg_io_last_error(). */
int fsg_snapshot_begin(fsg_session* s);
int fsg_snapshot_wait(fsg_session* s, double* rho, double* u);
int fsg_write_vtk(fsg_session* s, const char* path, const double origin[3]);
const char* fsg_io_last_error(void);
int fsg_write_vtk_fields(const char* path, const int dims[3], const double* rho, const double* u,
                         double dx, double dt, double rho_phys, const double origin[3]);
int fsg_format_full(double v, char* buf, int size);
typedef struct fsg_csv fsg_csv;
int fsg_csv_open(const char* path, int n_cols, const char* const* columns, fsg_csv** out);
int fsg_csv_write_row(fsg_csv* h, int n, const double* values);
int fsg_csv_close(fsg_csv* h);

/* ---- measurement ---------------------------------------------------------
 * When enabled, every step is bracketed with CUDA events on the session
 * stream (the marker kernel and the banded collide/stream kernel overlap, so
 * the step is one interval); read back the accumulated device time (ms) and
 * the number of timed steps. */
int fsg_profile_enable(fsg_session* s, int enable);
int fsg_profile_read(fsg_session* s, double* step_ms, int* steps);

/* ---- batched envs (BASELINE config 5) ------------------
 * n_envs (<= 64) independent sessions of one fp32 configuration sharing one
 * stream; fsg_batch_step_async steps every env with ONE marker launch and ONE
 * collide/stream launch.  Env e is an ordinary session handle
 * (fsg_batch_session): set its frame and markers and read it back with the
 * per-session calls; it is destroyed with the batch. */
typedef struct fsg_batch fsg_batch;
int fsg_batch_create(const fsg_config* cfg, int n_envs, fsg_batch** out);
int fsg_batch_destroy(fsg_batch* b);
fsg_session* fsg_batch_session(fsg_batch* b, int env);
int fsg_batch_step_async(fsg_batch* b);
int fsg_batch_step(fsg_batch* b, fsg_status* statuses /* n_envs, nullable */);
/* Every env with one skinned body (fsg_set_skin on each env): the frames
 * (n_envs, NULL: keep) and poses (n_envs) in, one batched step, every env's
 * status, tau_ext (concatenated) and CouplingStats (7 per env) out -- the RL
 * rollout loop's per-step exchange in one call. */
int fsg_batch_step_skinned(fsg_batch* b, const fsg_frame_state* frames, const fsg_body_pose* poses,
                           fsg_status* statuses, double* tau_ext, double* stats);
/* The whole CoupledSession::step (session.hpp:87-176) for every env, on the
 * device: env e's skinned body is robot e of the dyn handle (n_envs equal;
 * fsg_dyn_set_rest called).  Its pose comes from the robot state (forward
 * kinematics + BoneTransforms, no host round trip), the coupled fluid step
 * runs, and its tau_ext feeds the robot step (buoyancy_gravity_forces +
 * integrate, session.hpp:169-175) in the same stream.  Up: frames (NULL:
 * keep) and actuation [n_envs * n_joints]; down: statuses, robot flags and
 * the post-step robot states (each nullable).  tau_ext never leaves the
 * device between the fluid and the robot step.  dt and rho_fluid must be the
 * envs' cfg.dt and cfg.rho (the reference integrates with the session's
 * units, session.hpp:171-174).  With following on (fsg_batch_set_follow)
 * frames must be NULL: each env's frame is its FrameFollower's state, which
 * the call advances after the robot step, recentring the env's lattice when
 * the robot's COM leaves the threshold (session.hpp:177-195) -- the
 * reference's whole CoupledSession::step with the robot on the device. */
int fsg_batch_step_dynamic(fsg_batch* b, fsg_dyn* d, const fsg_frame_state* frames,
                           const double* actuation, double rho_fluid, const double* g_hydro,
                           double dt, int substeps, fsg_status* statuses, int* flags,
                           fsg_joint_state* states);
/* Frame following inside fsg_batch_step_dynamic: one FrameFollower per env in
 * the envs' cfg.frame_mode (not NONE) with time_constant (frame_time_constant,
 * session.hpp:17) and recenter_threshold_cells (session.hpp:18).
 * time_constant <= 0 turns following off (frames are then the caller's). */
int fsg_batch_set_follow(fsg_batch* b, double time_constant, double recenter_threshold_cells);
/* center_frame_on_robot for every env (session.hpp:210-221): each follower is
 * reset to its robot's current base position and yaw; the envs' frames too. */
int fsg_batch_center_frames(fsg_batch* b, fsg_dyn* d);
/* the recentre shifts the last fsg_batch_step_dynamic applied, [3 * n_envs]
 * (0 where the env's robot stayed inside the threshold) */
int fsg_batch_last_shifts(const fsg_batch* b, int* shifts);

/* ---- z-slab halo exchange ------------------------------
 * A slab session (cfg.z_offset / cfg.nz_global) owns planes [z_offset,
 * z_offset + dims[2]) of a global grid plus one halo plane per side.  Per
 * step, the 5 populations that cross each z face (5 * nx * ny elements per
 * face) go to the neighbour slab:
 *   fsg_step_async  updates the two boundary planes first, packs them into the
 *                   session's send buffers, then updates the interior planes;
 *   fsg_halo_begin  makes comm_stream wait until those planes are packed;
 *                   the caller moves send_hi -> upper neighbour's recv_lo and
 *                   send_lo -> lower neighbour's recv_hi on comm_stream (NCCL
 *                   or peer copies), overlapping the interior update;
 *   fsg_halo_end    makes the session stream wait for comm_stream and unpacks
 *                   the received planes (have_lo/have_hi: a neighbour exists)
 *                   into the halo before the next step.
 * fsg_halo_pack/unpack are the unordered primitives on the current state
 * (caller buffers).  Sizes in bytes. */
size_t fsg_halo_bytes(fsg_session* s);
int fsg_halo_pack(fsg_session* s, void* d_send_lo, void* d_send_hi);
int fsg_halo_unpack(fsg_session* s, const void* d_recv_lo, const void* d_recv_hi);
int fsg_halo_buffers(fsg_session* s, void** d_send_lo, void** d_send_hi, void** d_recv_lo,
                     void** d_recv_hi);
int fsg_halo_begin(fsg_session* s, void* comm_stream);
int fsg_halo_end(fsg_session* s, void* comm_stream, int have_lo, int have_hi);

/* ---- z-slab peer transport: the halo exchange inside the library ---------
 * (fp32 slab sessions.)  Each rank exports a handle of its
 * slab session (CUDA IPC handles of its two distribution buffers and of two
 * 32-bit delivery counters, plus its geometry), moves the handles between
 * ranks by any means (MPI, torch.distributed, a file), and connects to its
 * lower and upper neighbours' handles (NULL at a closed global face).  From
 * then on fsg_step_async alone runs the sharded step, stream-ordered and
 * without host involvement: the interior planes; a stream wait until each
 * neighbour has delivered its previous step's planes; the two boundary
 * planes, whose collision kernel stores the 5 crossing populations of each
 * face straight into the neighbour's halo plane (NVLink peer memory); a
 * stream-ordered counter write into each neighbour.  No pack/unpack, no
 * NCCL on the data path; the fsg_halo_* calls are not used.
 * Contract: every rank connects (after all have exported) with its session
 * idle, all ranks then run the same sequence of steps, and a rank destroys
 * its session only after all ranks have synchronized (a barrier). */
#define FSG_PEER_HANDLE_BYTES 512
typedef struct {
  unsigned char bytes[FSG_PEER_HANDLE_BYTES];
} fsg_peer_handle;
int fsg_peer_export(fsg_session* s, fsg_peer_handle* out);
int fsg_peer_connect(fsg_session* s, const fsg_peer_handle* lower, const fsg_peer_handle* upper);
int fsg_peer_disconnect(fsg_session* s);

#ifdef __cplusplus
}
#endif
#endif /* FSG_H */
