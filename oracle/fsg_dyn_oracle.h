/* fsg_dyn_oracle.h -- TEST INFRASTRUCTURE ONLY: fp64 restatement of the
 * reference's articulated-body dynamics (fishsim/robot/dynamics.hpp), the
 * checker for the device robot step (include/fsg.h, fsg_dyn_*).  The POD
 * types are the boundary's own (fsg_robot, fsg_joint_state, fsg_body_pose). */
#ifndef FSG_DYN_ORACLE_H
#define FSG_DYN_ORACLE_H
#include "../include/fsg.h"

typedef struct {                           /* KinematicsCache (dynamics.hpp:14-21) */
  double E[FSG_DYN_MAX_LINKS][9];          /* x_up: rotation parent -> link   */
  double r[FSG_DYN_MAX_LINKS][3];          /* x_up: link origin in parent     */
  double R_world[FSG_DYN_MAX_LINKS][9];
  double p_world[FSG_DYN_MAX_LINKS][3];
  double v_body[FSG_DYN_MAX_LINKS][6];
  double omega_world[FSG_DYN_MAX_LINKS][3];
  double v_origin_world[FSG_DYN_MAX_LINKS][3];
} orc_kcache;

void orc_quat_to_R(const double* q, double* R);
void orc_angle_axis_R(double angle, const double* axis, double* R);
void orc_quat_exp(const double* w, double* q);
int orc_dyn_floating(const fsg_robot* r);
int orc_dyn_n_joints(const fsg_robot* r);
int orc_dyn_n_dofs(const fsg_robot* r);
int orc_dyn_dof_index(const fsg_robot* r, int i);
void orc_spatial_inertia(double mass, const double* com, const double* Ic, double* I);
void orc_forward_kinematics(const fsg_robot* r, const fsg_joint_state* st, orc_kcache* kc);
void orc_mass_matrix(const fsg_robot* r, const orc_kcache* kc, double* H);
void orc_bias_forces(const fsg_robot* r, const fsg_joint_state* st, const orc_kcache* kc,
                     const double* g, double* c);
int orc_internal_forces(const fsg_robot* r, const fsg_joint_state* st, const double* act, double* tau);
void orc_joint_limit_forces(const fsg_robot* r, const fsg_joint_state* st, double* tau);
int orc_llt_solve(int n, const double* M, const double* b, double* x);
int orc_forward_dynamics(const fsg_robot* r, const fsg_joint_state* st, const double* tau_int,
                         const double* tau_ext, const double* g, double* qdd);
void orc_accumulate_point_force(const fsg_robot* r, const orc_kcache* kc, int link,
                                const double* p, const double* f, double* tau);
void orc_buoyancy_gravity_forces(const fsg_robot* r, const orc_kcache* kc, double bladder_volume,
                                 double rho, const double* g, double* tau);
int orc_integrate(const fsg_robot* r, fsg_joint_state* st, const double* act, const double* tau_ext,
                  double dt, int substeps, const double* g);
int orc_robot_step(const fsg_robot* r, fsg_joint_state* st, double bladder_volume, const double* act,
                   const double* tau_ext, double rho, const double* g_hydro, double dt, int substeps,
                   const double* g);
double orc_mechanical_energy(const fsg_robot* r, const fsg_joint_state* st, const double* g);
void orc_dyn_pose(const fsg_robot* r, const fsg_joint_state* st, const double* rest_R,
                  const double* rest_p, fsg_body_pose* pose);
#endif
