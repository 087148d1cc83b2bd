/* fsg_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C, fp64 restatement of the reference's IB-LBM hot path
 * (FishGym, /root/reference/proj/include/fishsim, see each function's
 * file:line).  It is the CHECKER for the CUDA product path: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 *
 * Parity pinning: every function here is compared bit-for-bit against the
 * reference's own headers compiled unmodified into oracle/_ref/libfishref.so
 * (tests/test_oracle.py), and the golden fixtures in tests/golden/ were
 * produced by that same _ref build (tests/golden/make_golden.py).
 *
 * Layout conventions (lattice.hpp:83-90): cell = x + nx*(y + ny*z);
 * distributions direction-major f[i*n + cell]; vector fields AoS [3*cell+k].
 */
#ifndef FSG_ORACLE_H
#define FSG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* lattice.hpp:17-38 */
extern const int ORC_EX[19], ORC_EY[19], ORC_EZ[19];
extern const double ORC_W[19];

/* units.hpp:25-26 */
double orc_tau(double dx, double dt, double nu);

/* lattice.hpp:41-45 */
double orc_equilibrium_dir(int i, double rho, const double u[3]);
/* lattice.hpp:107-116 */
void orc_initialize(const int dims[3], const double* rho, const double* u, double* f);

/* solver.hpp:25-51 ; returns n_nonpositive_rho */
int orc_macroscopic(const int dims[3], const double* f, const double* F, double* rho, double* u);
/* solver.hpp:65-97 */
void orc_apply_open_boundary(const int dims[3], double* f);
/* solver.hpp:103-178 : reads fa, writes fb (then caller swaps), applies the
 * open boundary to fb when !periodic. */
void orc_collide_and_stream(const int dims[3], int periodic, double tau, const double* fa,
                            double* fb, const double* F, int* finite, double* min_f);
/* solver.hpp:181-200 */
double orc_total_mass(const int dims[3], const double* f);
void orc_total_momentum(const int dims[3], const double* f, double p[3]);

/* kernel.hpp:22-40, coupling.hpp:18-24 ; kernel 0 = Peskin4, 1 = Roma3 */
double orc_phi(int kernel, double r);
void orc_range(int kernel, double x, int* lo, int* hi);
int orc_marker_in_bounds(int kernel, const int dims[3], const double x[3]);
/* coupling.hpp:27-48 */
void orc_interpolate(int kernel, const int dims[3], const double* ufield, const double x[3],
                     double out[3]);
/* coupling.hpp:52-71 */
void orc_spread(int kernel, const int dims[3], double* F, const double x[3], const double f[3]);
/* coupling.hpp:80-85 ; wall 0 = Slip, 1 = NoSlip */
void orc_direct_forcing(const double ub[3], const double uf[3], const double n[3], double rho,
                        double area, double h, double dt, int wall, double out[3]);

/* Frame constants derived from a world-frame FrameState (frame.hpp:13-53).
 * q = (w,x,y,z).  R is row-major. */
typedef struct {
  double p[3], pd[3], pdd[3], q[4], omega[3], alpha[3];
} orc_frame_state;
typedef struct {
  double R[9];       /* rotation() = q.toRotationMatrix()           */
  double a0[3];      /* R^T pdd                                     */
  double omega_f[3]; /* R^T omega                                   */
  double alpha_f[3]; /* R^T alpha                                   */
} orc_frame_consts;
void orc_frame_consts_of(const orc_frame_state* fs, orc_frame_consts* fc);
/* frame.hpp:47-53 */
void orc_virtual_force(const orc_frame_consts* fc, const double x[3], const double u[3],
                       double out[3]);
/* frame.hpp:132-154 : dst <- src shifted, caller swaps; advances fs->p */
void orc_recenter(const int dims[3], double dx, const double* src, double* dst, const int shift[3],
                  orc_frame_state* fs);

/* Session: the fluid half of CoupledSession::step (session.hpp:94-166). */
typedef struct orc_session orc_session;
orc_session* orc_session_create(const int dims[3], double dx, double dt, double rho, double nu,
                                int periodic, int kernel, int wall, int frame_mode);
void orc_session_destroy(orc_session* s);
double* orc_session_f(orc_session* s);     /* current (post-stream) f, 19*n */
double* orc_session_force(orc_session* s); /* F from the last step, 3*n     */
double* orc_session_rho(orc_session* s);   /* bare macro of the last step   */
double* orc_session_u(orc_session* s);
void orc_session_set_frame(orc_session* s, const orc_frame_state* fs);
void orc_session_get_frame(orc_session* s, orc_frame_state* fs);
/* stats per body: fluid force[3], body force[3], power ; returns nonpos count */
int orc_session_step(orc_session* s, int n_bodies, const int64_t* body_offsets,
                     const double* points, const double* velocities, const double* normals,
                     const double* areas, double* force_world, int* valid, double* stats,
                     int* finite, double* min_f);
void orc_session_recenter(orc_session* s, const int shift[3]);

/* ---- skinned bodies ---------------------------------
 * Restated from skinning.hpp / sampling.hpp / dynamics.hpp, which need
 * dynamic-size Eigen (VectorXd/MatrixXd blocks, Ref, LLT) and so do not
 * compile against the fixed-size stand-in: parity of this restatement is
 * pinned by the reference's own property tests for these functions
 * (test_sampling.cpp:45-193, test_ib.cpp:215-249), restated in
 * tests/test_skin_oracle.py.  Layouts match fsg_skeleton / fsg_body_pose. */
typedef struct {
  int n_links, floating_base, n_dofs;
  int parent[12], dof_index[12];
  double axis[12][3];
} orc_skeleton;
typedef struct {
  double bone_R[12][9], bone_t[12][3], R_world[12][9], p_world[12][3], v_origin_world[12][3],
      omega_world[12][3];
} orc_body_pose;
/* update_samples (sampling.hpp:307-322): points, velocities, normals [3m];
 * weights [m][n_links] dense */
void orc_update_samples(const orc_skeleton* sk, const orc_body_pose* pose, int m,
                        const double* rest, const double* nrest, const double* weights,
                        double* pts, double* vel, double* nrm);
/* session.hpp:129-143 for one body: for every valid marker in ascending
 * order, accumulate_skinned_force(..., -f_world, tau) (skinning.hpp:147-156 ->
 * dynamics.hpp:216-233) and the CouplingStats sums.  tau [n_dofs] and
 * stats[7] are zeroed first (session.hpp:106-107). */
void orc_skin_tau(const orc_skeleton* sk, const orc_body_pose* pose, int m, const double* rest,
                  const double* weights, const double* fworld, const int* valid,
                  const double* vel, double* tau, double* stats);

/* EmpiricalBackend::step surface work for one robot (empirical.hpp:74-100):
 * update_samples, surface_force (empirical.hpp:25-30, skipped when
 * f.isZero(): every |f_c| <= 1e-12), accumulate_skinned_force with +f,
 * force on body and power; stats[0..2] (force on fluid) stay 0. */
void orc_empirical_step(const orc_skeleton* sk, const orc_body_pose* pose, int m,
                        const double* rest, const double* nrest, const double* weights,
                        const double* areas, double k, double* tau, double* stats);

#ifdef __cplusplus
}
#endif
#endif
